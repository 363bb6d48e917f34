"""Times the runtime's own TP all-reduce (mt_tp_allreduce_bf16 on the context's TP communicator) in
isolation. torchrun --nproc-per-node N tools/tp_ar_probe.py"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist

from paper_2201_11990_b200._native import lib
from paper_2201_11990_b200.runtime import Context

dist.init_process_group("gloo")
r, w = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(r)
obj = [Context.unique_id() if r == 0 else None]
dist.broadcast_object_list(obj, src=0)
ctx = Context(r)
ctx.init_comm(obj[0], w, r, tensor=w)
s = torch.cuda.current_stream()
for mb in (25, 50):
    n = int(mb * 2**20 / 2)
    x = torch.ones(n, dtype=torch.bfloat16, device="cuda")
    for _ in range(5):
        lib().mt_tp_allreduce_bf16(ctx._h, C.c_void_p(x.data_ptr()), n, C.c_void_p(s.cuda_stream))
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        lib().mt_tp_allreduce_bf16(ctx._h, C.c_void_p(x.data_ptr()), n, C.c_void_p(s.cuda_stream))
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 20
    if r == 0:
        print(f"runtime TP={w} {mb} MB: {t*1e3:.1f} us ({n*2/(t*1e-3)/1e9:.0f} GB/s algbw)", flush=True)
ctx.close()
