"""NVLink bytes of the layer's TP all-reduces, from the GPU's own NVLink data counters (NVML
NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX / _RX, KiB, summed over the active links) around K repeats of:

  fwd   : mt_layer_forward of a GPT-3-shape layer (TP=N): the fused row-parallel GEMM + NVLS all-reduce
          (fc2, and the projection when K = h/t >= 4096) / GEMM + standalone NVLS kernel (projection at
          TP >= 4) — two all-reduces of b*s*h bf16 per forward;
  nccl  : two ncclAllReduce of the same b*s*h bf16 buffer (the NCCL path the fused kernels replace).

Prints per-GPU bytes per all-reduce against the models: ring 2(t-1)/t * B each way; NVLink SHARP
(multimem.ld_reduce of this rank's 1/t + multimem.st of it) ~ B + B/t transmitted, B/t + B received.

    torchrun --nproc-per-node N tools/nvlink_probe.py [--hidden 12288] [--reps 10]
"""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2201_11990_b200 import planner as PL  # noqa: E402
from paper_2201_11990_b200._native import lib  # noqa: E402
from paper_2201_11990_b200.runtime import Context, Layer  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--hidden", type=int, default=12288)
ap.add_argument("--heads", type=int, default=96)
ap.add_argument("--seq", type=int, default=2048)
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()

dist.init_process_group("gloo")
r, w = dist.get_rank(), dist.get_world_size()
local = int(os.environ.get("LOCAL_RANK", r))
torch.cuda.set_device(local)
pynvml.nvmlInit()
dev = pynvml.nvmlDeviceGetHandleByIndex(local)
links = []
for link in range(18):
    try:
        if pynvml.nvmlDeviceGetNvLinkState(dev, link) == pynvml.NVML_FEATURE_ENABLED:
            links.append(link)
    except pynvml.NVMLError:
        pass


def counters():
    """(tx, rx) bytes summed over the active links."""
    tx = rx = 0
    for link in links:
        vals = pynvml.nvmlDeviceGetFieldValues(dev, [(pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, link),
                                                     (pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX, link)])
        tx += vals[0].value.ullVal
        rx += vals[1].value.ullVal
    return tx * 1024, rx * 1024


obj = [Context.unique_id() if r == 0 else None]
dist.broadcast_object_list(obj, src=0)
ctx = Context(local)
ctx.init_comm(obj[0], w, r, tensor=w)
s = torch.cuda.current_stream()
layer = Layer(ctx, PL.layer_desc(a.hidden, a.heads, a.seq, 1, tp_size=w, tp_rank=r))
layer.init_params(s)
M = a.seq
x = torch.randn(M, a.hidden, device="cuda").bfloat16()
y = torch.empty_like(x)
g = torch.randn(M, a.hidden, device="cuda").bfloat16() * 1e-3
dx = torch.empty_like(x)
B = M * a.hidden * 2  # bytes of one all-reduce buffer
for i in range(3):
    layer.forward(x.data_ptr(), y.data_ptr(), i, s)
    layer.backward(g.data_ptr(), dx.data_ptr(), i, s)
torch.cuda.synchronize()


def measure(fn, tag, n_ar):
    dist.barrier()
    torch.cuda.synchronize()
    t0, r0 = counters()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(a.reps):
        fn(i)
    e1.record()
    torch.cuda.synchronize()
    t1, r1 = counters()
    per = a.reps * n_ar
    tx, rx = (t1 - t0) / per, (r1 - r0) / per
    ring = 2 * (w - 1) / w * B
    res = [None] * w
    dist.all_gather_object(res, (tx, rx, e0.elapsed_time(e1) / a.reps))
    if r == 0:
        for rank, (tx_, rx_, ms) in enumerate(res):
            print(f"{tag} TP={w} rank {rank}: {tx_ / 1e6:.1f} MB tx, {rx_ / 1e6:.1f} MB rx per all-reduce of "
                  f"{B / 1e6:.1f} MB (ring model {ring / 1e6:.1f} each way; NVLS model {(B + B / w) / 1e6:.1f} tx / "
                  f"{(B / w + B) / 1e6:.1f} rx); {ms:.3f} ms per rep", flush=True)


measure(lambda i: (layer.forward(x.data_ptr(), y.data_ptr(), 100 + i, s),
                   layer.backward(g.data_ptr(), dx.data_ptr(), 100 + i, s)) and None, "fwd+bwd (2 fused/NVLS + 2 NCCL)", 4)
buf = torch.ones(M * a.hidden, dtype=torch.bfloat16, device="cuda")
measure(lambda i: [lib().mt_tp_allreduce_bf16(ctx._h, C.c_void_p(buf.data_ptr()), buf.numel(),
                                              C.c_void_p(s.cuda_stream)) for _ in range(2)], "nccl", 2)
# the forward alone: its saved activations are freed by a matching backward after the counters are read
fwd_ids = []


def fwd_only(i):
    layer.forward(x.data_ptr(), y.data_ptr(), 1000 + i, s)
    fwd_ids.append(1000 + i)


measure(fwd_only, "fwd (fused GEMM+NVLS, NVLS kernel)", 2)
for i in fwd_ids:
    layer.backward(g.data_ptr(), dx.data_ptr(), i, s)
torch.cuda.synchronize()
layer.close()
ctx.close()
