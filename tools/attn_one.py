"""Run the GPT-3-shape layer forward+backward a few times with the fused attention (ncu target)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("MT_ATTN_FUSED", "1")
from paper_2201_11990_b200 import planner as PL  # noqa: E402
from paper_2201_11990_b200.runtime import Context, Layer  # noqa: E402
ctx = Context(0)
L = Layer(ctx, PL.layer_desc(12288, 96, 2048, 1))
s = torch.cuda.current_stream()
L.init_params(s)
x = torch.randn(2048, 12288, device="cuda").bfloat16()
y, dx = torch.empty_like(x), torch.empty_like(x)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    L.forward(x.data_ptr(), y.data_ptr(), 0, s)
    L.backward(x.data_ptr(), dx.data_ptr(), 0, s)
torch.cuda.synchronize()
print("ok")
