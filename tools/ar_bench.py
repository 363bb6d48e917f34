"""NCCL all-reduce bandwidth probe (torch.distributed, same libnccl as the runtime).
torchrun --nproc-per-node N tools/ar_bench.py [MB]"""
import os
import sys

import torch
import torch.distributed as dist

dist.init_process_group("nccl")
r, w = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(r)
for mb in [float(x) for x in (sys.argv[1:] or ["12.5", "25", "50", "100"])]:
    n = int(mb * 2**20 / 2)
    x = torch.ones(n, dtype=torch.bfloat16, device="cuda")
    for _ in range(5):
        dist.all_reduce(x)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        dist.all_reduce(x)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 20
    if r == 0:
        algbw = n * 2 / (t * 1e-3) / 1e9
        print(f"N={w} {mb:6.1f} MB: {t*1e3:7.1f} us  algbw {algbw:6.0f} GB/s  busbw {algbw*2*(w-1)/w:6.0f} GB/s", flush=True)
dist.destroy_process_group()
