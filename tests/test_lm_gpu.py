"""Language-model stage (SURVEY.md §8f N3 wired into the 1F1B driver): token ids in, cross-entropy out.

The stage must run exactly the op sequence a user would compose by hand from the module-level C ABI
(embed -> layers -> tied head + CE -> layers backward -> embedding backward, per microbatch in 1F1B
order), so the comparison partner here is that manual composition on separate Layer / Vocab objects
with the same parameters (the modules themselves are checked against numpy / the CPU oracle in
test_vocab_gpu.py and test_layer_gpu.py). Tolerance: 1e-5 relative (the embedding-gradient
scatter-add uses float atomics, so the summation order may differ); the loss must match to 1e-6.
"""
import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402
from paper_2201_11990_b200 import planner as PL  # noqa: E402
from paper_2201_11990_b200.runtime import Context, Layer, Stage, Vocab, adam_defaults  # noqa: E402

pytestmark = pytest.mark.gpu

SEED = 20260919
V, H, HEADS, S, B = 1000, 256, 4, 128, 2


def rel(a, b):
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-30))


def vocab_params(seed=0, vpad=None):
    """Global bf16-representable vocab parameters (word table padded to vpad rows)."""
    rng = np.random.default_rng(seed)
    bf = lambda a: O.from_bf16_bits(O.to_bf16_bits(a))  # noqa: E731
    word = bf(rng.standard_normal((vpad, H)).astype(np.float32) * 0.02)
    pos = bf(rng.standard_normal((S, H)).astype(np.float32) * 0.02)
    g = bf(1 + rng.standard_normal(H).astype(np.float32) * 0.02)
    be = bf(rng.standard_normal(H).astype(np.float32) * 0.02)
    return [np.ascontiguousarray(O.to_bf16_bits(a)) for a in (word, pos, g, be)]


def make_vocab(ctx, tp=1, rank=0, seed=0):
    v = Vocab(ctx, V, H, S, B, tp, rank, 0.1, 1e-5, SEED)
    vpad, _, _ = v.padded()
    for i, bits in enumerate(vocab_params(seed, vpad)):
        v.set_param(i, bits.ctypes.data)
    return v


def token_batch(mb, seed=1):
    rng = np.random.default_rng(seed)
    tok = rng.integers(0, V, (mb, B * S)).astype(np.int32)
    tgt = np.roll(tok, -1, axis=1).copy()  # next-token targets
    return tok, tgt


def vocab_grads(v):
    _, _, vp = v.padded()
    out = []
    for i, n in enumerate((vp * H, S * H, H, H)):
        a = np.empty(n, np.float32)
        v.get_grad(i, a.ctypes.data)
        out.append(a)
    return out


def layer_grads(lay):
    out = []
    for i, p in enumerate(O.param_shapes(H)):
        a = np.empty(p[0] * p[1], np.float32)
        lay.get_grad(i, a.ctypes.data)
        out.append(a)
    return out


def test_lm_stage_matches_manual_composition():
    L, MB = 2, 2
    ctx = Context(0)
    s = torch.cuda.current_stream()
    d = PL.layer_desc(H, HEADS, S, B, seed=SEED)
    st = Stage(ctx, d, L, MB)
    st.init_params(L, s)
    voc = make_vocab(ctx)
    st.attach_vocab(voc)
    tok, tgt = token_batch(MB)
    tok_h, tgt_h = torch.from_numpy(tok).pin_memory(), torch.from_numpy(tgt).pin_memory()
    loss = st.train_step(tok_h.data_ptr(), tgt_h.data_ptr(), s)
    got_layers = [layer_grads(st.layer(i)) for i in range(L)]
    got_vocab = vocab_grads(voc)

    # manual composition on independent objects with the same parameters
    lays = [Layer(ctx, PL.layer_desc(H, HEADS, S, B, seed=SEED, layer_index=i)) for i in range(L)]
    for lay in lays:
        lay.init_params(s)
        lay.zero_grads(s)
    v2 = make_vocab(ctx)
    from paper_2201_11990_b200._native import check, lib
    sp = C.c_void_p(s.cuda_stream)
    check(lib().mt_vocab_zero_grads(v2._h, sp))
    check(lib().mt_vocab_set_loss_scale(v2._h, 1.0 / MB))  # the stage's batch mean
    loss_d = torch.zeros(1, device="cuda")
    acts = [torch.empty(B * S, H, dtype=torch.bfloat16, device="cuda") for _ in range(L + 1)]
    g0, g1 = (torch.empty(B * S, H, dtype=torch.bfloat16, device="cuda") for _ in range(2))
    tok_d, tgt_d = torch.from_numpy(tok).cuda(), torch.from_numpy(tgt).cuda()
    for mb in range(MB):
        tp_ = C.c_void_p(tok_d[mb].data_ptr())
        check(lib().mt_vocab_embed_forward(v2._h, tp_, C.c_void_p(acts[0].data_ptr()), mb, sp))
        for i, lay in enumerate(lays):
            lay.forward(acts[i].data_ptr(), acts[i + 1].data_ptr(), mb, s)
        check(lib().mt_vocab_head_loss(v2._h, C.c_void_p(acts[L].data_ptr()), C.c_void_p(tgt_d[mb].data_ptr()),
                                       C.c_void_p(acts[L].data_ptr()), C.c_void_p(loss_d.data_ptr()), sp))
        cur, nxt = acts[L], g0
        for lay in reversed(lays):
            lay.backward(cur.data_ptr(), nxt.data_ptr(), mb, s)
            cur, nxt = nxt, (g1 if nxt is g0 else g0)
        check(lib().mt_vocab_embed_backward(v2._h, tp_, C.c_void_p(cur.data_ptr()), mb, sp))
    torch.cuda.synchronize()
    want_loss = float(loss_d.item())
    assert abs(loss - want_loss) <= 1e-6 * abs(want_loss), (loss, want_loss)
    assert 0.9 * np.log(V) < loss < 1.1 * np.log(V)  # batch mean, ~uniform prediction at init
    for i, lay in enumerate(lays):
        for p, (a, b) in enumerate(zip(got_layers[i], layer_grads(lay))):
            assert rel(a, b) < 1e-5, (i, p, rel(a, b))
    for p, (a, b) in enumerate(zip(got_vocab, vocab_grads(v2))):
        assert rel(a, b) < 1e-5, (p, rel(a, b))
    assert np.abs(got_vocab[0]).max() > 0 and np.abs(got_vocab[1]).max() > 0

    # device-resident token path: same iteration, same loss
    loss_dev = torch.zeros(1, device="cuda")
    st.set_step(0)  # replay the host-input iteration (same dropout masks)
    st.train_step_dev(tok_d.data_ptr(), tgt_d.data_ptr(), loss_dev.data_ptr(), s)
    torch.cuda.synchronize()
    assert abs(float(loss_dev.item()) - loss) <= 1e-6 * abs(loss)
    for lay in lays:
        lay.close()
    v2.close()
    st.close()
    voc.close()
    ctx.close()


def test_lm_stage_requires_tokens_and_matching_shape():
    from paper_2201_11990_b200._native import ConfigError
    ctx = Context(0)
    st = Stage(ctx, PL.layer_desc(H, HEADS, S, B, seed=SEED), 1, 1)
    bad = Vocab(ctx, V, H, S, 2 * B, 1, 0, 0.1, 1e-5, SEED)  # micro_batch mismatch
    with pytest.raises(ConfigError):
        st.attach_vocab(bad)
    voc = make_vocab(ctx)
    st.attach_vocab(voc)
    with pytest.raises(ConfigError):
        st.train_step(None, None, torch.cuda.current_stream())
    st.close()
    bad.close()
    voc.close()
    ctx.close()


def test_lm_training_memorises_a_batch():
    """Fixed batch, AdamW with the recipe's constants at a constant lr: the cross-entropy must fall
    well below the uniform-prediction value ln(V) (end-to-end check that the embedding, the layers,
    the tied head and the optimizer all receive and apply consistent gradients)."""
    L, MB = 2, 2
    ctx = Context(0)
    s = torch.cuda.current_stream()
    st = Stage(ctx, PL.layer_desc(H, HEADS, S, B, seed=SEED, dropout_hidden=0.0, dropout_attn=0.0), L, MB)
    st.init_params(L, s)
    voc = Vocab(ctx, V, H, S, B, 1, 0, 0.0, 1e-5, SEED)
    vpad, _, _ = voc.padded()
    for i, bits in enumerate(vocab_params(0, vpad)):
        voc.set_param(i, bits.ctypes.data)
    st.attach_vocab(voc)
    tok, tgt = token_batch(MB, seed=3)
    tok_h, tgt_h = torch.from_numpy(tok).pin_memory(), torch.from_numpy(tgt).pin_memory()
    losses = []
    for step in range(1, 31):
        losses.append(st.train_step(tok_h.data_ptr(), tgt_h.data_ptr(), s))  # batch mean
        norm = st.optimizer_step(adam_defaults(lr=1e-3, step=step, weight_decay=0.0), s)
        assert np.isfinite(norm) and norm > 0
    assert losses[0] > 0.9 * np.log(V)
    assert losses[-1] < 0.5 * losses[0], losses
    # tied table changed (the optimizer covers the vocab parameters)
    _, _, vp = voc.padded()
    w = np.empty(vp * H, np.uint16)
    voc.get_param(0, w.ctypes.data)
    assert not np.array_equal(w, vocab_params(0, vpad)[0].reshape(-1)[: vp * H])
    st.close()
    voc.close()
    ctx.close()


def test_lm_stage_consumes_blend_feed_with_batch_ramp(tmp_path):
    """N4 end to end: a blend manifest with a growing global batch (4 then 8 samples at b=2 -> 2 then
    4 microbatches) feeds the language-model stage through mt_feed_fill + mt_stage_set_micro_batches.
    The 2-microbatch iteration of a stage created for 4 must equal a stage created for exactly 2
    (to 1e-6: the per-row cross-entropy is summed with float atomics)."""
    from paper_2201_11990_b200.feed import Feed, blend_manifest
    m = tmp_path / "blend_manifest.jsonl"
    blend_manifest(m, [("web", 0.6, list(range(50))), ("code", 0.4, list(range(900, 930)))], 2, 0,
                   shuffle=True, config_seed=5, batch_per_step=[4, 8])
    feed = Feed(m, V, S, B, 1, 0, seed=SEED)
    ctx = Context(0)
    s = torch.cuda.current_stream()
    voc = make_vocab(ctx)
    losses = {}
    for cap in (4, 2):
        st = Stage(ctx, PL.layer_desc(H, HEADS, S, B, seed=SEED), 1, cap)
        st.init_params(1, s)
        st.attach_vocab(voc)
        G, MB = feed.step_info(0)
        assert (G, MB) == (4, 2)
        tok = torch.zeros(cap, B * S, dtype=torch.int32).pin_memory()
        tgt = torch.zeros(cap, B * S, dtype=torch.int32).pin_memory()
        feed.fill(0, tok.data_ptr(), tgt.data_ptr(), cap)
        if cap == 4:
            from paper_2201_11990_b200._native import ConfigError
            with pytest.raises(ConfigError):
                st.set_micro_batches(5)
        st.set_micro_batches(MB)
        losses[cap] = st.train_step(tok.data_ptr(), tgt.data_ptr(), s)
        if cap == 4:  # the ramp's next step uses all four microbatches
            G1, MB1 = feed.step_info(1)
            assert (G1, MB1) == (8, 4)
            feed.fill(1, tok.data_ptr(), tgt.data_ptr(), cap)
            st.set_micro_batches(MB1)
            l1 = st.train_step(tok.data_ptr(), tgt.data_ptr(), s)
            assert np.isfinite(l1) and 0.9 * np.log(V) < l1 < 1.1 * np.log(V)
        st.close()
    assert abs(losses[4] - losses[2]) <= 1e-6 * losses[2], losses  # loss sum uses float atomics
    feed.close()
    voc.close()
    ctx.close()
