"""Achievable HBM bandwidth of a plain device copy at the row kernels' transfer sizes (the size-dependent
ceiling their roofline fraction should be read against; MEASURED_PEAKS.json's hbm_gbs is a 2 GiB copy).
CUDA events around one copy_, L2 flushed (256 MB write) before each, best of 20."""
import torch

flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
for mb in (25, 50, 100, 200, 400, 1024):
    n = mb * 1024 * 1024 // 2
    a = torch.randn(n, device="cuda").bfloat16()
    b = torch.empty_like(a)
    best = 1e9
    for _ in range(20):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        b.copy_(a)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"copy {mb} MB read + {mb} MB write: {best * 1e3:.1f} us = {2 * n * 2 / best / 1e6:.0f} GB/s", flush=True)
    best = 1e9
    for _ in range(20):  # write-only stream (what an epilogue-bound GEMM such as the score GEMM does)
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        b.fill_(0.5)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"fill {mb} MB: {best * 1e3:.1f} us = {n * 2 / best / 1e6:.0f} GB/s", flush=True)
