"""Run the fused attention forward / backward of one GPT-3-shape layer (96 heads, hd 128, s 2048) a few
times — a clean ncu target.   python tools/attn_one.py [fwd|bwd] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("MT_ATTN_FUSED", "1")
import torch  # noqa: E402

from paper_2201_11990_b200 import planner as PL  # noqa: E402
from paper_2201_11990_b200.runtime import Context, Layer  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "fwd"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
h, H, s_ = int(os.environ.get("H", 12288)), int(os.environ.get("HEADS", 96)), int(os.environ.get("SEQ", 2048))
ctx = Context(0)
lay = Layer(ctx, PL.layer_desc(h, H, s_, 1, seed=5))
st = torch.cuda.current_stream()
lay.init_params(st)
x = torch.randn(s_, h, device="cuda").bfloat16()
y, dx = torch.empty_like(x), torch.empty_like(x)
g = (torch.randn(s_, h, device="cuda") * 1e-2).bfloat16()
for i in range(reps):
    lay.forward(x.data_ptr(), y.data_ptr(), i, st)
    lay.backward(g.data_ptr(), dx.data_ptr(), i, st)
torch.cuda.synchronize()
print("ok", which, reps)
