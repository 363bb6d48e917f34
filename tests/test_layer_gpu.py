"""GPU parity of the tensor-sliced layer (forward + backward) against the CPU oracle.

The GPU path runs entirely through the C ABI of libmtnlg.so (mt_layer_forward / mt_layer_backward);
the oracle is oracle/layer_oracle.cpp on the same seeded bf16 inputs and parameters.

Tolerances, relative Frobenius error:
  vs bf16-emulated oracle : activations <= 5e-3, gradients <= 1e-2
  vs fp32 oracle          : activations <= 2e-2, gradients <= 3e-2
Dropout masks are bit-identical by construction (tests/test_oracle.py pins the mask definition).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402
from paper_2201_11990_b200 import planner as PL  # noqa: E402
from paper_2201_11990_b200.runtime import Context, Layer  # noqa: E402

pytestmark = pytest.mark.gpu

SEED = 20260808


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def bf16_tensor(a: np.ndarray) -> "torch.Tensor":
    bits = O.to_bf16_bits(a)
    return torch.from_numpy(bits.view(np.int16)).view(torch.bfloat16).cuda()


def to_np(t: "torch.Tensor") -> np.ndarray:
    return t.float().cpu().numpy()


CASES = [
    # hidden, heads, seq, micro_batch, dropout
    (256, 4, 128, 4, 0.1),     # BASELINE configs[0] shape (tiny GPT layer), hd = 64
    (256, 4, 128, 4, 0.0),
    (1024, 8, 256, 1, 0.1),    # hd = 128
    (640, 4, 256, 1, 0.1),     # hd = 160 (MT-NLG head size)
]


@pytest.mark.parametrize("fused", [True, False], ids=["flash_attn", "unfused_attn"])
@pytest.mark.parametrize("hidden,heads,seq,mb,p", CASES)
def test_layer_matches_oracle(hidden, heads, seq, mb, p, fused, monkeypatch):
    # the attention path is chosen at layer creation: fused tcgen05 flash attention, or score GEMM +
    # causal softmax + PV GEMM (both must match the oracle)
    monkeypatch.setenv("MT_ATTN_FUSED", "1" if fused else "0")
    ctx = Context(0)
    desc = PL.layer_desc(hidden, heads, seq, mb, dropout_hidden=p, dropout_attn=p, seed=SEED, layer_index=3)
    layer = Layer(ctx, desc)
    params = O.init_params(hidden, SEED, 3)
    keep = []
    for i, prm in enumerate(params):
        bits = np.ascontiguousarray(O.to_bf16_bits(prm))
        keep.append(bits)
        layer.set_param(i, bits.ctypes.data)
    M = mb * seq
    x = O.normal(O.site_seed(SEED, "input", 0, 0), M, hidden)
    g = O.normal(O.site_seed(SEED, "grad", 0, 0), M, hidden, std=1e-2)
    xd, gd = bf16_tensor(x), bf16_tensor(g)
    yd = torch.empty_like(xd)
    dxd = torch.empty_like(xd)
    s = torch.cuda.current_stream()
    layer.forward(xd.data_ptr(), yd.data_ptr(), 0, s)
    layer.backward(gd.data_ptr(), dxd.data_ptr(), 0, s)
    torch.cuda.synchronize()
    y, dx = to_np(yd), to_np(dxd)
    grads = []
    for i, prm in enumerate(params):
        out = np.empty(prm.size, np.float32)
        layer.get_grad(i, out.ctypes.data)
        grads.append(out.reshape(prm.shape))

    for emu, tol_a, tol_g in ((True, 5e-3, 1e-2), (False, 2e-2, 3e-2)):
        ol = O.OracleLayer(hidden, heads, seq, mb, 1, dropout_hidden=p, dropout_attn=p, seed=SEED, layer_index=3,
                           bf16_emulate=emu, params=params)
        y_ref = ol.forward(x)
        dx_ref = ol.backward(g)
        assert rel(y, y_ref) < tol_a, ("y", emu, rel(y, y_ref))
        assert rel(dx, dx_ref) < tol_a * 2, ("dx", emu, rel(dx, dx_ref))
        for i, name in enumerate(O.PARAM_NAMES):
            assert rel(grads[i], ol.grads[i]) < tol_g, (name, emu, rel(grads[i], ol.grads[i]))
    layer.close()
    ctx.close()


@pytest.mark.parametrize("env", [{"MT_ATTN_BWD_WG": "1"}, {"MT_HIDDEN_KEEP": "0"}, {"MT_ATTN_GROUP_HEADS": "0"},
                                 {"MT_ATTN_GROUP_HEADS": "3", "MT_ATTN_FWD_GROUP_HEADS": "3"},
                                 {"MT_ATTN_FWD_BALANCED": "1"}, {"MT_ATTN_FWD_BALANCED": "0"}],
                         ids=["one_softmax_warpgroup", "rehash_hidden_dropout", "ungrouped_order", "groups_of_3",
                              "balanced_pairs", "adjacent_pairs"])
def test_runtime_switch_variants_match_oracle(env, monkeypatch):
    """The non-default variants behind the runtime switches against the oracle: one
    softmax warpgroup in the fused backward kernels, the backward re-hashing the hidden-dropout mask
    instead of reading the forward's keep bytes, and other launch-order groupings of the attention
    kernels (including a last, partial group: 8 heads in groups of 3)."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    test_layer_matches_oracle(1024, 8, 256, 1, 0.1, True, monkeypatch)


def _layer_outputs(hidden, heads, seq, mb, p):
    ctx = Context(0)
    layer = Layer(ctx, PL.layer_desc(hidden, heads, seq, mb, dropout_hidden=p, dropout_attn=p, seed=SEED,
                                     layer_index=3))
    for i, prm in enumerate(O.init_params(hidden, SEED, 3)):
        bits = np.ascontiguousarray(O.to_bf16_bits(prm))
        layer.set_param(i, bits.ctypes.data)
    M = mb * seq
    xd = bf16_tensor(O.normal(O.site_seed(SEED, "input", 0, 0), M, hidden))
    gd = bf16_tensor(O.normal(O.site_seed(SEED, "grad", 0, 0), M, hidden, std=1e-2))
    yd, dxd = torch.empty_like(xd), torch.empty_like(xd)
    s = torch.cuda.current_stream()
    layer.forward(xd.data_ptr(), yd.data_ptr(), 0, s)
    layer.backward(gd.data_ptr(), dxd.data_ptr(), 0, s)
    torch.cuda.synchronize()
    grads = []
    for i, shp in enumerate(O.param_shapes(hidden)):
        out = np.empty(int(np.prod(shp)), np.float32)
        layer.get_grad(i, out.ctypes.data)
        grads.append(out)
    res = (yd.view(torch.int16).cpu().numpy(), dxd.view(torch.int16).cpu().numpy(), grads)
    layer.close()
    ctx.close()
    return res


@pytest.mark.parametrize("env", [{"MT_HIDDEN_KEEP": "0"}, {"MT_ATTN_FWD_GROUP_HEADS": "3"},
                                 {"MT_ATTN_FWD_BALANCED": "1"}],
                         ids=["rehashed_hidden_mask", "forward_launch_groups", "forward_balanced_pairs"])
def test_switch_variants_are_bit_identical(env, monkeypatch):
    """Variants that must not change a single bit: the backward's hidden-dropout mask read from the
    forward's keep bytes vs re-hashed from the counter-based stream, and the forward attention's launch
    order. Deterministic path (MT_ATTN_BWD2=0: no dQ atomics), so every output and gradient is compared
    bitwise."""
    monkeypatch.setenv("MT_ATTN_BWD2", "0")
    monkeypatch.setenv("MT_ATTN_FWD_BALANCED", "0")
    base = _layer_outputs(1024, 8, 256, 1, 0.1)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    var = _layer_outputs(1024, 8, 256, 1, 0.1)
    assert np.array_equal(base[0], var[0]) and np.array_equal(base[1], var[1])
    for i, (a, b) in enumerate(zip(base[2], var[2])):
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), O.PARAM_NAMES[i]


@pytest.mark.parametrize("hidden,heads,seq,mb,attn_saved", [(1024, 8, 256, 1, True), (512, 8, 512, 2, True),
                                                             (640, 4, 256, 1, False)],
                         ids=["hd128", "hd64_two_rows", "hd160"])
def test_saved_dropout_keep_bits_are_bit_exact(hidden, heads, seq, mb, attn_saved):
    """The keep bits the kernels draw on the device and save for the backward — attention dropout
    (two-tile fused forward, hd <= 128: one bit per causal score) and both hidden dropouts
    (bias-dropout-residual kernels: one byte per 8 elements) — equal, bit for bit, the mask definition
    restated in numpy (tests/test_oracle.py keep_mask, pinned there against the native definition).
    The hd-160 forward does not save attention bits (its backward re-hashes them)."""
    from .test_oracle import keep_mask
    p, mbid, layer_index = 0.1, 5, 3
    ctx = Context(0)
    layer = Layer(ctx, PL.layer_desc(hidden, heads, seq, mb, dropout_hidden=p, dropout_attn=p, seed=SEED,
                                     layer_index=layer_index))
    layer.init_params(torch.cuda.current_stream())
    M = mb * seq
    xd = bf16_tensor(O.normal(O.site_seed(SEED, "input", 0, 0), M, hidden))
    yd = torch.empty_like(xd)
    layer.forward(xd.data_ptr(), yd.data_ptr(), mbid, torch.cuda.current_stream())
    # attention: words [b][heads][s][s / 32]; compare the causal 128-column blocks the forward writes
    if not attn_saved:
        with pytest.raises(PL.ConfigError):
            layer.dropout_keep_bits(mbid, 0, mb * heads * seq * seq // 8)
    words = np.frombuffer(layer.dropout_keep_bits(mbid, 0, mb * heads * seq * seq // 8), np.uint32) \
        if attn_saved else None
    words = words.reshape(mb, heads, seq, seq // 32) if attn_saved else None
    ref = keep_mask(O.site_seed(SEED, "attn.probs", layer_index, mbid), mb * heads * seq * seq, p)
    ref_words = np.packbits(ref.reshape(mb, heads, seq, seq // 32, 32)[..., ::-1], axis=-1,
                            bitorder="big").view(">u4").astype(np.uint32).reshape(mb, heads, seq, seq // 32)
    for i in range(seq if attn_saved else 0):
        nw = (i // 128 + 1) * 4  # words of the causal blocks of row i
        assert np.array_equal(words[:, :, i, :nw], ref_words[:, :, i, :nw]), ("attention row", i)
    # hidden dropout: bytes [b*s][h/8], bit j of byte v = element 8v + j
    for which, site in ((1, "attn.out"), (2, "mlp.out")):
        got = np.frombuffer(layer.dropout_keep_bits(mbid, which, M * hidden // 8), np.uint8)
        want = np.packbits(keep_mask(O.site_seed(SEED, site, layer_index, mbid), M * hidden, p).reshape(-1, 8),
                           axis=-1, bitorder="little").reshape(-1)
        assert np.array_equal(got, want), site
    gd = torch.zeros_like(xd)
    dxd = torch.empty_like(xd)
    layer.backward(gd.data_ptr(), dxd.data_ptr(), mbid, torch.cuda.current_stream())
    torch.cuda.synchronize()
    layer.close()
    ctx.close()


def test_device_init_matches_oracle_streams():
    """mt_layer_init_params draws, shard by shard, the same global tensors as the oracle's host
    generator (so TP=t and TP=1 runs start from identical weights)."""
    hidden, heads = 256, 4
    ctx = Context(0)
    ref = O.init_params(hidden, SEED, 5)
    for tp in (1, 2):
        for r in range(tp):
            desc = PL.layer_desc(hidden, heads, 128, 1, tp_size=tp, tp_rank=r, seed=SEED, layer_index=5)
            layer = Layer(ctx, desc)
            layer.init_params(torch.cuda.current_stream())
            torch.cuda.synchronize()
            for i in range(len(ref)):
                _, (r0, c0), (nr, nc) = PL.param_shard(desc, i)
                got = np.empty(nr * nc, np.uint16)
                layer.get_param(i, got.ctypes.data)
                want = O.to_bf16_bits(ref[i][r0:r0 + nr, c0:c0 + nc]).ravel()
                # device (libdevice) and host (glibc) log/sin/cos may differ in the last double ulp;
                # after rounding to bf16 that flips at most a handful of values by one ulp.
                diff = np.abs(got.astype(np.int32) - want.astype(np.int32))
                assert diff.max() <= 1 and (diff > 0).mean() < 1e-3, (tp, r, i)
            layer.close()
    ctx.close()


def test_layer_rejects_bad_config():
    ctx = Context(0)
    with pytest.raises(PL.ConfigError):
        Layer(ctx, PL.layer_desc(256, 3, 128, 1))  # heads do not divide hidden
    with pytest.raises(PL.ConfigError):
        Layer(ctx, PL.layer_desc(256, 4, 128, 1, tp_size=8, tp_rank=0))  # heads % TP
    ctx.close()


@pytest.mark.parametrize("shape", [(1024, 8, 256, 2, "auto"), (1024, 8, 256, 2, "2"), (4096, 32, 2048, 2, "auto")],
                         ids=["h1024", "h1024_split_rows", "h4096_splitk"])
@pytest.mark.parametrize("fused", [False, True], ids=["unfused_attn", "flash_attn"])
def test_activation_recompute_is_bit_identical(fused, shape, monkeypatch):
    """with recompute the backward re-runs the forward (same dropout masks) — the
    outputs, input gradients and parameter gradients must be bit-identical to the stored path. The
    h=4096, M=4096 case runs fc2 forward / fc1 dgrad (K = 16384) through the split-K tail (256 pair
    tiles = 3 waves + 34), whose fixed-order partial sum keeps the re-run bit-identical."""
    monkeypatch.setenv("MT_ATTN_FUSED", "1" if fused else "0")
    # the one-kernel fused backward accumulates dQ with fp32 atomics (order varies between runs): the
    # bit-identity check uses the deterministic dK/dV + dQ kernel pair
    monkeypatch.setenv("MT_ATTN_BWD2", "0")
    hidden, heads, seq, mb, split = shape
    monkeypatch.setenv("MT_ROWS_SPLIT", split)  # "2": the row kernels split each row over a CTA pair
    out = []
    for rc in (False, True):
        ctx = Context(0)
        lay = Layer(ctx, PL.layer_desc(hidden, heads, seq, mb, seed=SEED, layer_index=1))
        lay.set_recompute(rc)
        params = O.init_params(hidden, SEED, 1)
        for i, p in enumerate(params):
            b = np.ascontiguousarray(O.to_bf16_bits(p))
            lay.set_param(i, b.ctypes.data)
        x = bf16_tensor(O.normal(O.site_seed(SEED, "input", 0, 0), mb * seq, hidden))
        g = bf16_tensor(O.normal(O.site_seed(SEED, "grad", 0, 0), mb * seq, hidden, std=1e-2))
        y, dx = torch.empty_like(x), torch.empty_like(x)
        s = torch.cuda.current_stream()
        lay.zero_grads(s)
        for m in range(2):  # two microbatches in flight, like a pipeline stage
            lay.forward(x.data_ptr(), y.data_ptr(), m, s)
        for m in range(2):
            lay.backward(g.data_ptr(), dx.data_ptr(), m, s)
        torch.cuda.synchronize()
        grads = []
        for i, p in enumerate(params):
            a = np.empty(p.size, np.float32)
            lay.get_grad(i, a.ctypes.data)
            grads.append(a)
        out.append((y.cpu().view(torch.int16).numpy(), dx.cpu().view(torch.int16).numpy(), grads))
        lay.close()
        ctx.close()
    (y0, dx0, g0), (y1, dx1, g1) = out
    assert (y0 == y1).all() and (dx0 == dx1).all()
    for a, b in zip(g0, g1):
        assert (a == b).all()


def test_dropout_masks_follow_the_training_step():
    """masks are keyed by curator::step_seed(seed, step) so they change every iteration; a
    layer at step 3 matches the oracle run with that seed, and differs from step 0."""
    hidden, heads, seq, mb = 256, 4, 128, 2
    ctx = Context(0)
    layer = Layer(ctx, PL.layer_desc(hidden, heads, seq, mb, dropout_hidden=0.1, dropout_attn=0.1, seed=SEED,
                                     layer_index=2))
    params = O.init_params(hidden, SEED, 2)
    keep = [np.ascontiguousarray(O.to_bf16_bits(p)) for p in params]
    for i, b in enumerate(keep):
        layer.set_param(i, b.ctypes.data)
    x = O.normal(O.site_seed(SEED, "input", 0, 0), mb * seq, hidden)
    g = O.normal(O.site_seed(SEED, "grad", 0, 0), mb * seq, hidden, std=1e-2)
    xd, gd = bf16_tensor(x), bf16_tensor(g)
    s = torch.cuda.current_stream()
    ys = {}
    for step in (0, 3):
        yd, dxd = torch.empty_like(xd), torch.empty_like(xd)
        layer.set_step(step)
        layer.zero_grads(s)
        layer.forward(xd.data_ptr(), yd.data_ptr(), 0, s)
        layer.set_step(99)  # the backward replays the forward's masks whatever the current step
        layer.backward(gd.data_ptr(), dxd.data_ptr(), 0, s)
        torch.cuda.synchronize()
        ol = O.OracleLayer(hidden, heads, seq, mb, 1, dropout_hidden=0.1, dropout_attn=0.1,
                           seed=O.step_seed(SEED, step), layer_index=2, bf16_emulate=True, params=params)
        y_ref, dx_ref = ol.forward(x), ol.backward(g)
        assert rel(to_np(yd), y_ref) < 5e-3 and rel(to_np(dxd), dx_ref) < 1e-2, step
        ys[step] = to_np(yd)
    assert rel(ys[3], ys[0]) > 1e-2
    assert O.step_seed(SEED, 0) == SEED and O.step_seed(SEED, 3) != SEED
    layer.close()
    ctx.close()


@pytest.mark.parametrize("split", ["1", "2"], ids=["whole_rows", "split_rows"])
def test_row_kernels_whole_and_split_rows_match_oracle(split, monkeypatch):
    """The LayerNorm / bias-dropout-residual(+LN) / LayerNorm-backward row kernels in both layouts:
    whole rows per CTA, and each row's columns split over a cluster of two CTAs (the layout of the
    LayerNorm-carrying kernels at h > 12288, forced here at h = 1024 with MT_ROWS_SPLIT=2), whose LayerNorm statistics combine the
    halves' (mean, M2) over DSMEM. Both match the oracle; they agree with each other to fp32 rounding of
    the statistics."""
    hidden, heads, seq, mb, p = 1024, 8, 128, 2, 0.1
    params = O.init_params(hidden, SEED, 4)
    x = O.normal(O.site_seed(SEED, "input", 0, 0), mb * seq, hidden)
    g = O.normal(O.site_seed(SEED, "grad", 0, 0), mb * seq, hidden, std=1e-2)
    res = {}
    for mode in ("1", split):
        monkeypatch.setenv("MT_ROWS_SPLIT", mode)
        ctx = Context(0)
        layer = Layer(ctx, PL.layer_desc(hidden, heads, seq, mb, dropout_hidden=p, dropout_attn=p, seed=SEED,
                                         layer_index=4))
        keep = [np.ascontiguousarray(O.to_bf16_bits(prm)) for prm in params]
        for i, b in enumerate(keep):
            layer.set_param(i, b.ctypes.data)
        xd, gd = bf16_tensor(x), bf16_tensor(g)
        yd, dxd = torch.empty_like(xd), torch.empty_like(xd)
        s = torch.cuda.current_stream()
        layer.forward(xd.data_ptr(), yd.data_ptr(), 0, s)
        layer.backward(gd.data_ptr(), dxd.data_ptr(), 0, s)
        torch.cuda.synchronize()
        grads = []
        for i, prm in enumerate(params):
            out = np.empty(prm.size, np.float32)
            layer.get_grad(i, out.ctypes.data)
            grads.append(out.reshape(prm.shape))
        res[mode] = (to_np(yd), to_np(dxd), grads)
        layer.close()
        ctx.close()
    y, dx, grads = res[split]
    ol = O.OracleLayer(hidden, heads, seq, mb, 1, dropout_hidden=p, dropout_attn=p, seed=SEED, layer_index=4,
                       bf16_emulate=True, params=params)
    y_ref, dx_ref = ol.forward(x), ol.backward(g)
    assert rel(y, y_ref) < 5e-3 and rel(dx, dx_ref) < 1e-2
    for i, name in enumerate(O.PARAM_NAMES):
        assert rel(grads[i], ol.grads[i]) < 1e-2, name
    y1, dx1, g1 = res["1"]
    assert rel(y, y1) < 2e-3 and rel(dx, dx1) < 2e-3
    for a, b in zip(grads, g1):  # bf16 rounding flips of the LN outputs reach the small bias gradients
        assert rel(a, b) < 5e-3
