"""NVLS all-reduce throughput probe over the runtime's symmetric buffer (mt_ctx_nvls_probe).
torchrun --nproc-per-node N tools/nvls_probe.py"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["MT_TP_FUSED"] = "1"
import torch
import torch.distributed as dist

from paper_2201_11990_b200 import planner as PL
from paper_2201_11990_b200._native import check, lib
from paper_2201_11990_b200.runtime import Context, Layer

dist.init_process_group("gloo")
r, w = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(r)
obj = [Context.unique_id() if r == 0 else None]
dist.broadcast_object_list(obj, src=0)
ctx = Context(r)
ctx.init_comm(obj[0], w, r, tensor=w)
lay = Layer(ctx, PL.layer_desc(12288, 96, 2048, 1, tp_size=w, tp_rank=r))
elems = 2048 * 12288
for strided in (0, 1):
    for ctas in (16, 32, 64, 148):
        us = C.c_double()
        check(lib().mt_ctx_nvls_probe(ctx._h, elems, 12288, strided, ctas, 20, C.byref(us)))
        if r == 0:
            print(f"TP={w} {'tiles' if strided else 'contig'} ctas={ctas}: {us.value:.1f} us "
                  f"({elems * 2 / (us.value * 1e-6) / 1e9:.0f} GB/s algbw)", flush=True)
lay.close()
ctx.close()
