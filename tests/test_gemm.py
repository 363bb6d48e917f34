"""tcgen05 GEMM (csrc/gemm_sm100.cu) against a torch fp32 reference of the same contraction.

Tolerance: bf16 output rounding (2^-8 relative) plus fp32 accumulation-order differences;
checked as relative Frobenius error <= 1e-2 and elementwise |err| <= 2e-2 * max|ref| + 1e-3.
"""
import ctypes as C

import pytest

torch = pytest.importorskip("torch")

from paper_2201_11990_b200 import _native as N  # noqa: E402

pytestmark = pytest.mark.gpu


def _gemm(a, b, d, m, n, k, *, a_mn=False, b_mn=False, batch=1, lda=None, ldb=None, ldd=None,
          abs_=0, bbs=0, dbs=0, alpha=1.0, epi=N.EPI_STORE_BF16, causal=0, bias=None, aux=None, ld_aux=0, bn=0,
          ws=None, max_ctas=0):
    args = N.GemmArgs()
    args.a, args.b, args.d = a.data_ptr(), b.data_ptr(), d.data_ptr()
    args.lda = lda if lda is not None else (m if a_mn else k)
    args.ldb = ldb if ldb is not None else (n if b_mn else k)
    args.ldd = ldd if ldd is not None else n
    args.a_batch_stride, args.b_batch_stride, args.d_batch_stride = abs_, bbs, dbs
    args.a_mn_major, args.b_mn_major = int(a_mn), int(b_mn)
    args.m, args.n, args.k, args.batch = m, n, k, batch
    args.alpha, args.epilogue, args.causal = alpha, epi, causal
    args.bias = bias.data_ptr() if bias is not None else None
    args.aux = aux.data_ptr() if aux is not None else None
    args.ld_aux, args.block_n, args.max_ctas = ld_aux, bn, max_ctas
    if ws is not None:
        args.workspace, args.workspace_bytes = ws.data_ptr(), ws.numel()
    rc = N.lib().mt_gemm(C.byref(args), C.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == 0, rc
    torch.cuda.synchronize()


def _close(out, ref, tol=1e-2):
    out, ref = out.float(), ref.float()
    rel = (out - ref).norm() / ref.norm().clamp_min(1e-30)
    assert rel < tol, f"rel fro err {rel:.3e}"
    assert (out - ref).abs().max() <= 2e-2 * ref.abs().max() + 1e-3


@pytest.mark.parametrize("a_mn", [False, True])
@pytest.mark.parametrize("b_mn", [False, True])
@pytest.mark.parametrize("bn", [64, 128, 160, 192, 256])
@pytest.mark.parametrize("mnk", [(256, 512, 256), (296, 328, 200), (128, 160, 64)])
def test_gemm_majors(a_mn, b_mn, bn, mnk):
    m, n, k = mnk
    g = torch.Generator(device="cuda").manual_seed(1)
    A = torch.randn(m, k, device="cuda", generator=g).bfloat16()
    B = torch.randn(n, k, device="cuda", generator=g).bfloat16()
    a_store = A.t().contiguous() if a_mn else A
    b_store = B.t().contiguous() if b_mn else B
    D = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    _gemm(a_store, b_store, D, m, n, k, a_mn=a_mn, b_mn=b_mn, bn=bn)
    _close(D, A.float() @ B.float().t())


def test_gemm_epilogues():
    m, n, k = 512, 384, 320
    A = torch.randn(m, k, device="cuda").bfloat16()
    B = torch.randn(n, k, device="cuda").bfloat16() * 0.1
    bias = torch.randn(n, device="cuda").bfloat16()
    ref = A.float() @ B.float().t()
    D = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    _gemm(A, B, D, m, n, k, bias=bias)
    _close(D, ref + bias.float())
    pre = torch.empty_like(D)
    _gemm(A, B, D, m, n, k, bias=bias, epi=N.EPI_BIAS_GELU, aux=pre, ld_aux=n)
    _close(pre, ref + bias.float())
    _close(D, torch.nn.functional.gelu(pre.float(), approximate="tanh"))
    # GeLU backward: D = acc * gelu'(pre)
    x = pre.float().requires_grad_(True)
    torch.nn.functional.gelu(x, approximate="tanh").backward(torch.ones_like(x))
    _gemm(A, B, D, m, n, k, epi=N.EPI_GELU_BWD, aux=pre, ld_aux=n)
    _close(D, ref * x.grad)
    # fp32 store and accumulate
    F = torch.zeros(m, n, device="cuda", dtype=torch.float32)
    _gemm(A, B, F, m, n, k, epi=N.EPI_STORE_F32, alpha=0.5)
    _close(F, 0.5 * ref, 1e-5)
    _gemm(A, B, F, m, n, k, epi=N.EPI_ACCUM_F32)
    _close(F, 1.5 * ref, 1e-5)


def test_gemm_batched_strided_heads():
    # attention-style: qkv [s, heads, 3, hd]; S_h = Q_h K_h^T
    s, H, hd = 256, 3, 160
    qkv = torch.randn(s, H, 3, hd, device="cuda").bfloat16()
    S = torch.empty(H, s, s, device="cuda", dtype=torch.bfloat16)
    _gemm(qkv[:, :, 0], qkv[:, :, 1], S, s, s, hd, batch=H, lda=3 * H * hd, ldb=3 * H * hd, ldd=s,
          abs_=3 * hd, bbs=3 * hd, dbs=s * s, alpha=0.125)
    q = qkv[:, :, 0].float().permute(1, 0, 2)
    kk = qkv[:, :, 1].float().permute(1, 0, 2)
    _close(S, 0.125 * q @ kk.transpose(1, 2))
    # P V with V MN-major (hd contiguous), output into ctx [s, H*hd]
    P = torch.randn(H, s, s, device="cuda").bfloat16()
    ctx = torch.empty(s, H * hd, device="cuda", dtype=torch.bfloat16)
    _gemm(P, qkv[:, :, 2], ctx, s, hd, s, batch=H, b_mn=True, lda=s, ldb=3 * H * hd, ldd=H * hd,
          abs_=s * s, bbs=3 * hd, dbs=hd)
    v = qkv[:, :, 2].float().permute(1, 0, 2)
    _close(ctx.view(s, H, hd).permute(1, 0, 2), P.float() @ v)


@pytest.mark.parametrize("causal", [1, 2, 3])
def test_gemm_causal_modes(causal):
    s, k = 512, 128
    if causal == 1:
        A = torch.randn(s, k, device="cuda").bfloat16()
        B = torch.randn(s, k, device="cuda").bfloat16()
        D = torch.zeros(s, s, device="cuda", dtype=torch.bfloat16)
        _gemm(A, B, D, s, s, k, causal=1, bn=128)
        ref = A.float() @ B.float().t()
        mask = torch.ones(s, s, device="cuda", dtype=torch.bool).tril()
        _close(D[mask], ref[mask])
        return
    P = torch.randn(s, s, device="cuda")
    P = (P.tril() if causal == 2 else P.triu()).bfloat16()
    V = torch.randn(s, k, device="cuda").bfloat16()
    D = torch.empty(s, k, device="cuda", dtype=torch.bfloat16)
    _gemm(P, V, D, s, k, s, b_mn=True, causal=causal)
    _close(D, P.float() @ V.float())


@pytest.mark.parametrize("epi", [N.EPI_STORE_BF16, N.EPI_ACCUM_F32, N.EPI_BIAS_GELU])
@pytest.mark.parametrize("max_ctas", [0, 132, 40])
def test_gemm_split_k_tail(epi, max_ctas):
    """Shapes whose last wave is partial take the split-K tail path (partials + last-arriver reduce);
    the tail is split only for K >= 256 k-blocks (16384). The last arriver sums the splits' partials in
    a fixed order, so repeated launches are bit-identical."""
    m, n, k = 2048, 12288, 16384
    A = torch.randn(m, k, device="cuda").bfloat16()
    B = (torch.randn(n, k, device="cuda") * 0.05).bfloat16()
    bias = torch.randn(n, device="cuda").bfloat16()
    ws = torch.zeros(64 << 20, dtype=torch.uint8, device="cuda")
    ref = A.float() @ B.float().t()
    outs = []
    for _ in range(3):  # later launches check the counters were reset and the sum order is fixed
        if epi == N.EPI_ACCUM_F32:
            D = torch.ones(m, n, device="cuda")
            _gemm(A, B, D, m, n, k, epi=epi, ws=ws, max_ctas=max_ctas)
            _close(D, ref + 1.0, 1e-4)
        elif epi == N.EPI_BIAS_GELU:
            D = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
            pre = torch.empty_like(D)
            _gemm(A, B, D, m, n, k, epi=epi, bias=bias, aux=pre, ld_aux=n, ws=ws, max_ctas=max_ctas)
            _close(pre, ref + bias.float())
            _close(D, torch.nn.functional.gelu(pre.float(), approximate="tanh"))
        else:
            D = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
            _gemm(A, B, D, m, n, k, ws=ws, max_ctas=max_ctas)
            _close(D, ref)
        outs.append(D.clone())
    assert int(ws[: 64 * 1024].sum()) == 0  # counters left zeroed
    for o in outs[1:]:
        assert torch.equal(o.view(torch.int16) if o.dtype == torch.bfloat16 else o.view(torch.int32),
                           outs[0].view(torch.int16) if o.dtype == torch.bfloat16 else outs[0].view(torch.int32))




def test_gemm_dynamic_scheduler_matches_static():
    """With a workspace the GEMM hands tiles out dynamically (ticket counter in the workspace, raster
    order, per-pair mbarrier ring); without one it walks them round-robin. Every tile's arithmetic is
    the same either way, so for shapes without a split-K tail the outputs are bit-identical. A sequence
    of launches of different tile counts (fewer tiles than CTA pairs, several waves, causal batched,
    fp32 n-fastest) sharing one workspace also checks that the counter resets itself after each
    launch."""
    g = torch.Generator(device="cuda").manual_seed(7)
    ws = torch.zeros(64 << 20, dtype=torch.uint8, device="cuda")
    cases = [
        dict(m=256, n=512, k=256),                                   # 4 pair tiles < 74 pairs
        dict(m=2048, n=12288, k=4096),                               # ~5 waves, m-fastest, bf16
        dict(m=6144, n=1536, k=2048, a_mn=True, b_mn=True, f32=True),  # n-fastest wgrad shape, fp32 out
        dict(m=1024, n=1024, k=128, batch=6, causal=1),              # causal score GEMM, batched heads
        dict(m=1024, n=128, k=1024, batch=6, causal=2),              # causal P V GEMM (k-range clipped)
        dict(m=640, n=4096, k=1024, bn=160),                         # single-CTA (non-pair) tiles
    ]
    for rep in range(2):
        for cs in cases:
            m, n, k = cs["m"], cs["n"], cs["k"]
            batch = cs.get("batch", 1)
            a_mn, b_mn = cs.get("a_mn", False), cs.get("b_mn", False)
            A = torch.randn(batch, k, m, device="cuda", generator=g).bfloat16() if a_mn else \
                torch.randn(batch, m, k, device="cuda", generator=g).bfloat16()
            B = torch.randn(batch, k, n, device="cuda", generator=g).bfloat16() if b_mn else \
                torch.randn(batch, n, k, device="cuda", generator=g).bfloat16()
            dt = torch.float32 if cs.get("f32") else torch.bfloat16
            epi = N.EPI_STORE_F32 if cs.get("f32") else N.EPI_STORE_BF16
            outs = []
            for w in (None, ws):
                D = torch.zeros(batch, m, n, device="cuda", dtype=dt)
                _gemm(A, B, D, m, n, k, a_mn=a_mn, b_mn=b_mn, batch=batch, abs_=A[0].numel(), bbs=B[0].numel(),
                      dbs=D[0].numel(), epi=epi, causal=cs.get("causal", 0), bn=cs.get("bn", 0), ws=w)
                outs.append(D)
            view = torch.int32 if dt == torch.float32 else torch.int16
            assert torch.equal(outs[0].view(view), outs[1].view(view)), (rep, cs)
            assert int(ws[: 64 * 1024].sum()) == 0, (rep, cs)  # the ticket counter reset itself
