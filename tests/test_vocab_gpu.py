"""Vocab-parallel embedding + tied LM head + vocab-parallel cross-entropy on the
GPU against a numpy fp32 restatement (same seeded inputs, same dropout mask definition).

Tolerances: embedding output 5e-3 relative (bf16 storage), loss 2e-3 relative, gradients 2e-2
relative Frobenius (bf16 logit gradients).
"""
import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402
from paper_2201_11990_b200._native import VocabDesc, check, lib  # noqa: E402
from paper_2201_11990_b200.runtime import Context  # noqa: E402

SEED = 20260808
M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(z):
    z = (z + np.uint64(0x9E3779B97F4A7C15)) & M64
    z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & M64
    z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & M64
    return z ^ (z >> np.uint64(31))


def keep_mask(site, n, p):
    th = 0 if p <= 0 else int(round(p * 65536))
    idx = np.arange(n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        bits = splitmix64((np.uint64(site) + (idx >> np.uint64(2)) * np.uint64(0x9E3779B97F4A7C15)) & M64)
    return ((bits >> (np.uint64(16) * (idx & np.uint64(3)))) & np.uint64(0xFFFF)) >= np.uint64(th)


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-30))


def bf(a):
    return O.from_bf16_bits(O.to_bf16_bits(a))


def dev_bf16(a):
    return torch.from_numpy(O.to_bf16_bits(a).view(np.int16)).view(torch.bfloat16).cuda()


def reference(V, h, s, b, p, word, pos, g, be, tokens, targets, y, dx):
    M = b * s
    site = O.site_seed(SEED, "embed.dropout", 0, 0)
    keep = keep_mask(site, M * h, p).reshape(M, h)
    x = bf(word[tokens] + pos[np.arange(M) % s])
    x = x * keep / (1 - p)
    yf = y.astype(np.float64)
    mu = yf.mean(1, keepdims=True)
    var = ((yf - mu) ** 2).mean(1, keepdims=True)
    rs = 1 / np.sqrt(var + 1e-5)
    xh = (yf - mu) * rs
    yn = bf(xh * g + be)
    logits = yn.astype(np.float64) @ word[:V].T.astype(np.float64)
    mx = logits.max(1, keepdims=True)
    lse = mx[:, 0] + np.log(np.exp(logits - mx).sum(1))
    loss = float((lse - logits[np.arange(M), targets]).mean())
    sm = np.exp(logits - lse[:, None])
    sm[np.arange(M), targets] -= 1
    dl = bf(sm / M)
    dyn = dl @ word[:V].astype(np.float64)
    gg = dyn * g
    dy = rs * (gg - gg.mean(1, keepdims=True) - xh * (gg * xh).mean(1, keepdims=True))
    dword = np.zeros_like(word, dtype=np.float64)
    dword[:V] = dl.T @ yn.astype(np.float64)
    gx = dx * keep / (1 - p)
    np.add.at(dword, tokens, gx)
    dpos = np.zeros((s, h))
    np.add.at(dpos, np.arange(M) % s, gx)
    return x, loss, dy, dword, dpos, (dyn * xh).sum(0), dyn.sum(0)


@pytest.mark.gpu
@pytest.mark.parametrize("V", [1000, 1152])
def test_vocab_embedding_head_cross_entropy(V):
    h, s, b, p = 256, 128, 2, 0.1
    M = b * s
    ctx = Context(0)
    d = VocabDesc(V, h, s, b, 1, 0, p, 1e-5, SEED)
    hv = C.c_void_p()
    check(lib().mt_vocab_create(ctx._h, C.byref(d), C.byref(hv)))
    vpad, v0, vp = C.c_int64(), C.c_int64(), C.c_int64()
    check(lib().mt_vocab_padded(hv, C.byref(vpad), C.byref(v0), C.byref(vp)))
    assert vpad.value % 128 == 0 and vpad.value >= V and vp.value == vpad.value
    rng = np.random.default_rng(0)
    word = bf(rng.standard_normal((vpad.value, h)).astype(np.float32) * 0.05)
    pos = bf(rng.standard_normal((s, h)).astype(np.float32) * 0.02)
    g = bf(1 + rng.standard_normal(h).astype(np.float32) * 0.02)
    be = bf(rng.standard_normal(h).astype(np.float32) * 0.02)
    for i, a in enumerate((word, pos, g, be)):
        bits = np.ascontiguousarray(O.to_bf16_bits(a))
        check(lib().mt_vocab_set_param(hv, i, bits.ctypes.data))
    tokens = rng.integers(0, V, M).astype(np.int32)
    targets = rng.integers(0, V, M).astype(np.int32)
    y = bf(rng.standard_normal((M, h)).astype(np.float32))
    dxh = bf(rng.standard_normal((M, h)).astype(np.float32) * 1e-2)
    st = torch.cuda.current_stream()
    tok_d, tgt_d = torch.from_numpy(tokens).cuda(), torch.from_numpy(targets).cuda()
    x_d = torch.empty(M, h, dtype=torch.bfloat16, device="cuda")
    y_d, dy_d, dx_d = dev_bf16(y), torch.empty(M, h, dtype=torch.bfloat16, device="cuda"), dev_bf16(dxh)
    loss_d = torch.zeros(1, device="cuda")
    s_ = C.c_void_p(st.cuda_stream)
    check(lib().mt_vocab_zero_grads(hv, s_))
    check(lib().mt_vocab_embed_forward(hv, C.c_void_p(tok_d.data_ptr()), C.c_void_p(x_d.data_ptr()), 0, s_))
    check(lib().mt_vocab_head_loss(hv, C.c_void_p(y_d.data_ptr()), C.c_void_p(tgt_d.data_ptr()),
                                   C.c_void_p(dy_d.data_ptr()), C.c_void_p(loss_d.data_ptr()), s_))
    check(lib().mt_vocab_embed_backward(hv, C.c_void_p(tok_d.data_ptr()), C.c_void_p(dx_d.data_ptr()), 0, s_))
    torch.cuda.synchronize()
    x_ref, loss_ref, dy_ref, dword_ref, dpos_ref, dg_ref, db_ref = reference(V, h, s, b, p, word, pos, g, be, tokens,
                                                                             targets, y, dxh)
    assert rel(x_d.float().cpu().numpy(), x_ref) < 5e-3
    assert abs(float(loss_d.item()) - loss_ref) / loss_ref < 2e-3, (loss_d.item(), loss_ref)
    assert rel(dy_d.float().cpu().numpy(), dy_ref) < 2e-2
    grads = []
    for i, n in enumerate((vpad.value * h, s * h, h, h)):
        a = np.empty(n, np.float32)
        check(lib().mt_vocab_get_grad(hv, i, a.ctypes.data_as(C.POINTER(C.c_float))))
        grads.append(a)
    assert rel(grads[0].reshape(vpad.value, h), dword_ref) < 2e-2
    if vpad.value > V:
        assert np.abs(grads[0].reshape(vpad.value, h)[V:]).max() == 0.0  # padded rows never touched
    assert rel(grads[1].reshape(s, h), dpos_ref) < 1e-4
    assert rel(grads[2], dg_ref) < 2e-2 and rel(grads[3], db_ref) < 2e-2
    lib().mt_vocab_destroy(hv)
    ctx.close()
