"""Optimizer step: fused AdamW + global grad-norm clipping + curator::lr_at,
checked against a numpy restatement; lr schedule and recipe constants pinned to the reference.

CPU part (no GPU): the recipe defaults come from curator::TrainingRecipe (reference
planner.hpp:39-53) and the lr from curator::lr_at (planner.cpp:59-70, golden-pinned elsewhere).
"""
import numpy as np
import pytest

from paper_2201_11990_b200 import planner as PL
from paper_2201_11990_b200.runtime import adam_defaults


def test_recipe_defaults_match_reference_training_recipe():
    d = adam_defaults()
    assert d.lr < 0 and d.step == 1
    assert d.beta1 == pytest.approx(0.9) and d.beta2 == pytest.approx(0.95)
    assert d.eps == pytest.approx(1e-8) and d.grad_clip == pytest.approx(1.0) and d.weight_decay == pytest.approx(0.1)


def numpy_adamw(w, g, m, v, lr, b1, b2, eps, wd, step, clip, decay):
    coef = min(1.0, clip / (np.sqrt(sum(float((x.astype(np.float64) ** 2).sum()) for x in g)) + 1e-6)) if clip > 0 else 1.0
    out = []
    for wi, gi, mi, vi, di in zip(w, g, m, v, decay):
        gi = gi * np.float32(coef)
        mi = b1 * mi + (1 - b1) * gi
        vi = b2 * vi + (1 - b2) * gi * gi
        upd = (mi / (1 - b1 ** step)) / (np.sqrt(vi / (1 - b2 ** step)) + eps)
        if di:
            wi = wi - lr * wd * wi
        wi = wi - lr * upd
        out.append((wi, mi, vi))
    return out, coef


@pytest.mark.gpu
def test_layer_adam_step_matches_numpy():
    torch = pytest.importorskip("torch")
    from oracle import oracle as O
    from paper_2201_11990_b200.runtime import Context, Layer
    seed, h, H, s = 20260808, 256, 4, 128
    ctx = Context(0)
    lay = Layer(ctx, PL.layer_desc(h, H, s, 2, seed=seed))
    params = O.init_params(h, seed, 0)
    for i, p in enumerate(params):
        b = np.ascontiguousarray(O.to_bf16_bits(p))
        lay.set_param(i, b.ctypes.data)
    dev = lambda a: torch.from_numpy(O.to_bf16_bits(a).view(np.int16)).view(torch.bfloat16).cuda()  # noqa
    x = dev(O.normal(O.site_seed(seed, "input", 0, 0), 2 * s, h))
    g = dev(O.normal(O.site_seed(seed, "grad", 0, 0), 2 * s, h, std=0.5))
    y, dx = torch.empty_like(x), torch.empty_like(x)
    st = torch.cuda.current_stream()
    lay.zero_grads(st)
    lay.forward(x.data_ptr(), y.data_ptr(), 0, st)
    lay.backward(g.data_ptr(), dx.data_ptr(), 0, st)
    torch.cuda.synchronize()
    grads = []
    for i, p in enumerate(params):
        a = np.empty(p.size, np.float32)
        lay.get_grad(i, a.ctypes.data)
        grads.append(a.reshape(p.shape))
    tokens = 5e8
    desc = adam_defaults(tokens_seen=tokens, step=1, grad_clip=0.05)  # small clip: the clipping path is exercised
    norm = lay.adam_step(desc, st)
    want_norm = np.sqrt(sum(float((a.astype(np.float64) ** 2).sum()) for a in grads))
    assert norm == pytest.approx(want_norm, rel=1e-4)
    lr = PL.lr_at(tokens)
    decay = [i in (2, 4, 8, 10) for i in range(12)]
    want, coef = numpy_adamw([p.astype(np.float32) for p in params], grads, [np.zeros_like(p) for p in params],
                             [np.zeros_like(p) for p in params], lr, 0.9, 0.95, 1e-8, 0.1, 1, 0.05, decay)
    assert coef < 1.0
    for i, p in enumerate(params):
        mst, m, v = (np.empty(p.size, np.float32) for _ in range(3))
        lay.optimizer_state(i, mst.ctypes.data, m.ctypes.data, v.ctypes.data)
        w_want, m_want, v_want = want[i]
        np.testing.assert_allclose(m.reshape(p.shape), m_want, rtol=1e-5, atol=1e-12)
        np.testing.assert_allclose(v.reshape(p.shape), v_want, rtol=1e-4, atol=1e-16)
        np.testing.assert_allclose(mst.reshape(p.shape), w_want, rtol=1e-6, atol=1e-7)
        bits = np.empty(p.size, np.uint16)
        lay.get_param(i, bits.ctypes.data)
        assert (bits == O.to_bf16_bits(mst)).all()  # bf16 weights are the rounded masters
    lay.close()
    ctx.close()
