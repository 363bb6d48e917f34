"""Tiny end-to-end workload for compute-sanitizer (memcheck / racecheck / synccheck): one small layer
forward + backward through the C ABI on both attention paths (unfused and tcgen05 flash), a stage
iteration with host inputs, and a split-K GEMM — every hand-written kernel family of the path
(tcgen05 GEMM incl. split-K tail and pair tiles, TMA row kernels, softmax, dropout/residual, column
reductions, flash attention fwd/bwd, MSE loss). Exits 0 when every call returned status 0.

    compute-sanitizer --tool racecheck python tools/sanitize_tiny.py
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2201_11990_b200 import _native as N  # noqa: E402
from paper_2201_11990_b200 import planner as PL  # noqa: E402
from paper_2201_11990_b200.runtime import Context, Layer, Stage  # noqa: E402

torch.cuda.set_device(0)
s = torch.cuda.current_stream()
for fused in ("0", "1"):
    os.environ["MT_ATTN_FUSED"] = fused
    ctx = Context(0)
    lay = Layer(ctx, PL.layer_desc(512, 4, 256, 2, dropout_hidden=0.1, dropout_attn=0.1, seed=7))
    lay.init_params(s)
    x = torch.randn(512, 512, device="cuda").bfloat16()
    y, dx = torch.empty_like(x), torch.empty_like(x)
    g = (torch.randn(512, 512, device="cuda") * 1e-2).bfloat16()
    lay.forward(x.data_ptr(), y.data_ptr(), 0, s)
    lay.backward(g.data_ptr(), dx.data_ptr(), 0, s)
    torch.cuda.synchronize()
    assert torch.isfinite(dx.float()).all()
    lay.close()
    ctx.close()
    print(f"layer fwd+bwd (MT_ATTN_FUSED={fused}) ok", flush=True)
os.environ["MT_ATTN_FUSED"] = "0"
ctx = Context(0)
st = Stage(ctx, PL.layer_desc(256, 4, 128, 2, seed=9), 2, 2)
st.init_params(2, s)
xh = torch.randn(2, 256, 256).bfloat16().pin_memory()
th = torch.randn(2, 256, 256).bfloat16().pin_memory()
loss = st.train_step(xh.data_ptr(), th.data_ptr(), s)
assert loss == loss and loss > 0
st.close()
ctx.close()
print(f"stage iteration ok (loss {loss:.4f})", flush=True)
# split-K tail GEMM (K >= 16384, partial last wave) with the zeroed workspace
m, n, k = 512, 12288, 16384  # 96 pair tiles = 74 + a 22-tile tail split 3 ways
A = torch.randn(m, k, device="cuda").bfloat16()
B = (torch.randn(n, k, device="cuda") * 0.05).bfloat16()
D = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
ws = torch.zeros(64 << 20, dtype=torch.uint8, device="cuda")
a = N.GemmArgs()
a.a, a.b, a.d = A.data_ptr(), B.data_ptr(), D.data_ptr()
a.lda, a.ldb, a.ldd = k, k, n
a.m, a.n, a.k, a.batch, a.alpha, a.epilogue = m, n, k, 1, 1.0, N.EPI_STORE_BF16
a.workspace, a.workspace_bytes = ws.data_ptr(), ws.numel()
assert N.lib().mt_gemm(C.byref(a), C.c_void_p(s.cuda_stream)) == 0
torch.cuda.synchronize()
print("split-K GEMM ok", flush=True)
print("SANITIZE_TINY_OK")
