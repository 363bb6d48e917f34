"""CPU oracle self-pinning (no GPU): torch-autograd cross-check of the layer restatement,
TP=t == TP=1 equivalence, dropout-mask definition, seeded streams.

The reference has no implementation of the layer (parity unpinned upstream); these
tests pin the oracle itself before it is used to check the GPU kernels.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.nn.functional as F  # noqa: E402

from oracle import oracle as O  # noqa: E402

SEED = 20260808
M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(z):
    z = (z + np.uint64(0x9E3779B97F4A7C15)) & M64
    z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & M64
    z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & M64
    return z ^ (z >> np.uint64(31))


def keep_mask(site, n, p):
    """Vectorised restatement of include/curator/dropout.hpp (16-bit uniforms, 4 per SplitMix64 output)."""
    th = 0 if p <= 0 else int(round(p * 65536))
    idx = np.arange(n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        bits = splitmix64((np.uint64(site) + (idx >> np.uint64(2)) * np.uint64(0x9E3779B97F4A7C15)) & M64)
    u16 = (bits >> (np.uint64(16) * (idx & np.uint64(3)))) & np.uint64(0xFFFF)
    return u16 >= np.uint64(th)


def test_dropout_mask_definition_matches_native():
    site = O.site_seed(SEED, "attn.out", 7, 3)
    m = keep_mask(site, 4096, 0.1)
    native = np.array([O.lib().or_dropout_keep(site, i, int(round(0.1 * 65536))) for i in range(4096)], bool)
    assert (m == native).all()
    assert abs(1 - m.mean() - 0.1) < 0.02


def torch_layer(x, params, hidden, heads, seq, mb, p, layer_index, mbid=0):
    """fp32 autograd reference of the layer (same math, same masks)."""
    h, H, s, b = hidden, heads, seq, mb
    hd = h // H
    (g1, b1, wqkv, bqkv, wo, bo, g2, b2, w1, bf1, w2, bf2) = params
    sc = 1.0 / (1.0 - p)
    M = b * s
    m_attn = torch.from_numpy(keep_mask(O.site_seed(SEED, "attn.probs", layer_index, mbid), b * H * s * s, p)
                              .reshape(b, H, s, s)).float()
    m1 = torch.from_numpy(keep_mask(O.site_seed(SEED, "attn.out", layer_index, mbid), M * h, p).reshape(M, h)).float()
    m2 = torch.from_numpy(keep_mask(O.site_seed(SEED, "mlp.out", layer_index, mbid), M * h, p).reshape(M, h)).float()
    ln1 = F.layer_norm(x, (h,), g1.view(-1), b1.view(-1), 1e-5)
    qkv = (ln1 @ wqkv.t() + bqkv.view(-1)).view(b, s, H, 3, hd)
    q, k, v = (qkv[:, :, :, i].permute(0, 2, 1, 3) for i in range(3))
    S = (q @ k.transpose(-1, -2)) / np.sqrt(hd)
    causal = torch.ones(s, s, dtype=torch.bool).tril()
    S = S.masked_fill(~causal, float("-inf"))
    P = torch.softmax(S, -1) * m_attn * sc
    ctx = (P @ v).permute(0, 2, 1, 3).reshape(M, h)
    x1 = x + (ctx @ wo.t() + bo.view(-1)) * m1 * sc
    ln2 = F.layer_norm(x1, (h,), g2.view(-1), b2.view(-1), 1e-5)
    a = F.gelu(ln2 @ w1.t() + bf1.view(-1), approximate="tanh")
    return x1 + (a @ w2.t() + bf2.view(-1)) * m2 * sc


@pytest.mark.parametrize("p", [0.0, 0.1])
def test_oracle_fp32_matches_torch_autograd(p):
    hidden, heads, seq, mb = 128, 4, 64, 2
    params = O.init_params(hidden, SEED, 2)
    x = O.normal(O.site_seed(SEED, "input", 0, 0), mb * seq, hidden)
    g = O.normal(O.site_seed(SEED, "grad", 0, 0), mb * seq, hidden, std=1e-2)
    ol = O.OracleLayer(hidden, heads, seq, mb, 1, dropout_hidden=p, dropout_attn=p, seed=SEED, layer_index=2,
                       bf16_emulate=False, params=params)
    y = ol.forward(x)
    dx = ol.backward(g)
    tp = [torch.tensor(a, requires_grad=True) for a in params]
    tx = torch.tensor(x, requires_grad=True)
    ty = torch_layer(tx, tp, hidden, heads, seq, mb, p, 2)
    ty.backward(torch.tensor(g))
    np.testing.assert_allclose(y, ty.detach().numpy(), rtol=1e-4, atol=1e-4)
    np.testing.assert_allclose(dx, tx.grad.numpy(), rtol=1e-3, atol=1e-5)
    for i, name in enumerate(O.PARAM_NAMES):
        ref = tp[i].grad.numpy()
        err = np.linalg.norm(ol.grads[i] - ref) / max(np.linalg.norm(ref), 1e-30)
        assert err < 1e-4, (name, err)


@pytest.mark.parametrize("tp", [2, 4])
def test_oracle_tensor_parallel_equals_single(tp):
    """TP=t (per-shard partials summed = the emulated all-reduce) == TP=1 in fp32."""
    hidden, heads, seq, mb = 128, 4, 64, 2
    params = O.init_params(hidden, SEED, 1)
    x = O.normal(O.site_seed(SEED, "input", 0, 0), mb * seq, hidden)
    g = O.normal(O.site_seed(SEED, "grad", 0, 0), mb * seq, hidden, std=1e-2)
    outs = []
    for t in (1, tp):
        ol = O.OracleLayer(hidden, heads, seq, mb, t, dropout_hidden=0.1, dropout_attn=0.1, seed=SEED,
                           layer_index=1, bf16_emulate=False, params=params)
        outs.append((ol.forward(x), ol.backward(g), [gr.copy() for gr in ol.grads]))
    (y1, dx1, g1), (yt, dxt, gt) = outs
    np.testing.assert_allclose(yt, y1, rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(dxt, dx1, rtol=1e-4, atol=1e-7)
    for a, b in zip(gt, g1):
        np.testing.assert_allclose(a, b, rtol=1e-4, atol=1e-7)


def test_bf16_emulation_close_to_fp32():
    hidden, heads, seq, mb = 128, 4, 64, 1
    x = O.normal(O.site_seed(SEED, "input", 0, 0), mb * seq, hidden)
    ys = [O.OracleLayer(hidden, heads, seq, mb, bf16_emulate=e).forward(x) for e in (False, True)]
    err = np.linalg.norm(ys[0] - ys[1]) / np.linalg.norm(ys[0])
    assert 1e-5 < err < 1e-2


def test_normal_stream_statistics_and_determinism():
    a = O.normal(12345, 512, 512, round_bf16=False)
    b = O.normal(12345, 512, 512, round_bf16=False)
    assert (a == b).all()
    assert abs(a.mean()) < 0.01 and abs(a.std() - 1) < 0.01


def test_shard_init_matches_full_init_on_the_shard():
    """init_params(shard=...) draws exactly the shard's region of the full init (the rest zero)."""
    h, H, t = 256, 4, 2
    full = O.init_params(h, 7, 1)
    for r in range(t):
        part = O.init_params(h, 7, 1, shard=(H, t, r))
        for i in range(12):
            r0, c0, nr, nc = O.shard_region(i, h, H, t, r)
            assert np.array_equal(part[i][r0:r0 + nr, c0:c0 + nc], full[i][r0:r0 + nr, c0:c0 + nc])
            mask = np.ones_like(full[i], bool)
            mask[r0:r0 + nr, c0:c0 + nc] = False
            assert not part[i][mask].any()


def test_oracle_shard_mode_sums_to_the_full_layer_without_dropout():
    """Shard mode at TP=1 (one shard = the whole layer, nothing to all-reduce) is the full layer bit for bit;
    at TP>1 it is checked against the GPU's shard-only mode (tests/test_parity_bench.py)."""
    h, H, s = 256, 4, 64
    x = O.normal(O.site_seed(3, "input", 0, 0), s, h)
    g = O.normal(O.site_seed(3, "grad", 0, 0), s, h, std=1e-2)
    params = O.init_params(h, 3, 0)
    a = O.OracleLayer(h, H, s, 1, 1, seed=3, params=params)
    b = O.OracleLayer(h, H, s, 1, 1, seed=3, params=params, shard_rank=0)
    assert np.array_equal(a.forward(x), b.forward(x))
    assert np.array_equal(a.backward(g), b.backward(g))
    for ga, gb in zip(a.grads, b.grads):
        assert np.array_equal(ga, gb)
