"""Time the tcgen05 GEMM on the layer's shapes (CUDA events, L2 flushed between reps)."""
import ctypes as C
import sys
import torch
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_2201_11990_b200 import _native as N

def run(m, n, k, a_mn=False, b_mn=False, bn=0, epi=N.EPI_STORE_BF16, reps=10):
    A = torch.randn((k, m) if a_mn else (m, k), device="cuda").bfloat16()
    B = torch.randn((k, n) if b_mn else (n, k), device="cuda").bfloat16()
    D = torch.empty(m, n, device="cuda", dtype=torch.float32 if epi >= 3 else torch.bfloat16)
    a = N.GemmArgs(); a.a, a.b, a.d = A.data_ptr(), B.data_ptr(), D.data_ptr()
    a.lda = m if a_mn else k; a.ldb = n if b_mn else k; a.ldd = n
    a.a_mn_major, a.b_mn_major = int(a_mn), int(b_mn)
    a.m, a.n, a.k, a.batch, a.alpha, a.epilogue, a.block_n = m, n, k, 1, 1.0, epi, bn
    # the runtime's workspace (split-K tail counters / partials, dynamic tile scheduler)
    ws = torch.zeros(64 << 20, dtype=torch.uint8, device="cuda")
    a.workspace, a.workspace_bytes = ws.data_ptr(), ws.numel()
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        assert N.lib().mt_gemm(C.byref(a), s) == 0
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); N.lib().mt_gemm(C.byref(a), s); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort(); t = ts[len(ts) // 2]
    ref = (A.float().t() if a_mn else A.float()) @ (B.float() if b_mn else B.float().t())
    err = ((D.float() - ref).norm() / ref.norm()).item()
    tf = 2 * m * n * k / t / 1e9
    print(f"m={m} n={n} k={k} a_mn={a_mn} b_mn={b_mn} bn={bn} epi={epi}: {t*1e3:.1f} us  {tf:.0f} TFLOP/s  relerr={err:.2e}", flush=True)
    # torch (cuBLAS) for context
    if not a_mn and not b_mn:
        for _ in range(3): torch.matmul(A, B.t())
        e0.record()
        for _ in range(reps): torch.matmul(A, B.t())
        e1.record(); torch.cuda.synchronize()
        tc = e0.elapsed_time(e1) / reps
        print(f"   cuBLAS: {tc*1e3:.1f} us {2*m*n*k/tc/1e9:.0f} TFLOP/s", flush=True)

if __name__ == "__main__":
    run(2048, 36864, 12288)
    run(2048, 12288, 12288)
    run(2048, 49152, 12288)
    run(2048, 12288, 49152)
    run(2048, 12288, 36864, b_mn=True)          # dgrad
    run(36864, 12288, 2048, a_mn=True, b_mn=True, epi=N.EPI_ACCUM_F32)  # wgrad
    run(2048, 7680, 20480)                       # MT-NLG TP=8 QKV
    run(2048, 7680, 20480, bn=128)
    run(8192, 8192, 8192)
