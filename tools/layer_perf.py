"""Time one tensor-sliced layer fwd+bwd (single GPU, TP shard shapes) through the C ABI."""
import argparse
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2201_11990_b200 import planner as PL  # noqa: E402
from paper_2201_11990_b200.runtime import Context, Layer  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--hidden", type=int, default=12288)
ap.add_argument("--heads", type=int, default=96)
ap.add_argument("--seq", type=int, default=2048)
ap.add_argument("--tp", type=int, default=1)
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--profile", action="store_true")
a = ap.parse_args()
ctx = Context(0)
d = PL.layer_desc(a.hidden, a.heads, a.seq, 1, tp_size=a.tp, tp_rank=0)
L = Layer(ctx, d)
s = torch.cuda.current_stream()
L.init_params(s)
M = a.seq
x = torch.randn(M, a.hidden, device="cuda").bfloat16()
y = torch.empty_like(x)
g = torch.randn(M, a.hidden, device="cuda").bfloat16() * 1e-3
dx = torch.empty_like(x)
for _ in range(2):
    L.forward(x.data_ptr(), y.data_ptr(), 0, s); L.backward(g.data_ptr(), dx.data_ptr(), 0, s)
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
tf, tb = [], []
for _ in range(a.iters):
    e[0].record(); L.forward(x.data_ptr(), y.data_ptr(), 0, s); e[1].record()
    L.backward(g.data_ptr(), dx.data_ptr(), 0, s); e[2].record(); torch.cuda.synchronize()
    tf.append(e[0].elapsed_time(e[1])); tb.append(e[0].elapsed_time(e[2]))
h = a.hidden
flops = 72 * M * h * h * (1 + a.seq / (6 * h)) / a.tp
t = sorted(tb)[len(tb) // 2]
print(f"h={h} H={a.heads} s={a.seq} tp={a.tp}: fwd {sorted(tf)[len(tf)//2]:.2f} ms, fwd+bwd {t:.2f} ms, "
      f"{flops / t / 1e9:.0f} TFLOP/s/GPU, launches {L.launch_counts()}, finite={bool(torch.isfinite(dx.float()).all())}")
