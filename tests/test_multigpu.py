"""Multi-GPU parity (needs >= 2 GPUs; skipped otherwise): TP=2 layer, PP=2 1F1B stage pipeline, DP=2
gradient all-reduce — all through the C ABI with NCCL over NVLink, compared against the CPU oracle.

Tolerances as tests/test_layer_gpu.py (bf16-emulated oracle: activations 5e-3, gradients 1e-2 rel-Frobenius;
loss 5e-3 relative).
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

SEED = 20260808
H, HEADS, S, B = 512, 8, 256, 1


def _need(n):
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-30))


def _worker(rank, world, port, mode, q):
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_2201_11990_b200 import planner as PL
    from paper_2201_11990_b200.runtime import Context, Layer, Stage
    try:
        torch.cuda.set_device(rank)
        os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        obj = [Context.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ctx = Context(rank)
        s = torch.cuda.current_stream()
        out = {}
        if mode == "lm_pp":
            from tests import test_lm_gpu as LM
            from paper_2201_11990_b200.runtime import Vocab, adam_defaults  # noqa: F401
            MB = 4
            ctx.init_comm(obj[0], world, rank, tensor=1, pipeline=world, data=1, batch=LM.B * MB, micro_batches=MB)
            tok, tgt = LM.token_batch(MB)
            tok_h, tgt_h = torch.from_numpy(tok).pin_memory(), torch.from_numpy(tgt).pin_memory()

            def run(c, layers_here):
                st = Stage(c, PL.layer_desc(LM.H, LM.HEADS, LM.S, LM.B, seed=LM.SEED), 2, MB)
                st.init_params(layers_here, s)
                voc = LM.make_vocab(c)
                st.attach_vocab(voc)
                loss = st.train_step(tok_h.data_ptr(), tgt_h.data_ptr(), s)
                r = dict(loss=loss, layers=[LM.layer_grads(st.layer(i)) for i in range(layers_here)],
                         vocab=LM.vocab_grads(voc))
                r["norm"] = st.optimizer_step(adam_defaults(tokens_seen=2e9, step=1), s)
                st.close()
                voc.close()
                return r

            out["pp"] = run(ctx, 1)
            solo = Context(rank)  # the same model unpartitioned on this GPU (PP = 1)
            out["ref"] = run(solo, 2)
            solo.close()
        elif mode == "vocab":
            import ctypes as C
            from paper_2201_11990_b200._native import VocabDesc, check, lib
            ctx.init_comm(obj[0], world, rank, tensor=world)
            V, h, s_, b = 1000, 256, 128, 2
            M = s_ * b
            hv = C.c_void_p()
            check(lib().mt_vocab_create(ctx._h, C.byref(VocabDesc(V, h, s_, b, world, rank, 0.1, 1e-5, SEED)),
                                        C.byref(hv)))
            vpad, v0, vp = C.c_int64(), C.c_int64(), C.c_int64()
            check(lib().mt_vocab_padded(hv, C.byref(vpad), C.byref(v0), C.byref(vp)))
            rng = np.random.default_rng(0)
            bfr = lambda a: O.from_bf16_bits(O.to_bf16_bits(a))  # noqa
            word = bfr(rng.standard_normal((vpad.value, h)).astype(np.float32) * 0.05)
            pos = bfr(rng.standard_normal((s_, h)).astype(np.float32) * 0.02)
            g = bfr(1 + rng.standard_normal(h).astype(np.float32) * 0.02)
            be = bfr(rng.standard_normal(h).astype(np.float32) * 0.02)
            for i, a in enumerate((word, pos, g, be)):
                bits = np.ascontiguousarray(O.to_bf16_bits(a))
                check(lib().mt_vocab_set_param(hv, i, bits.ctypes.data))
            tokens = rng.integers(0, V, M).astype(np.int32)
            targets = rng.integers(0, V, M).astype(np.int32)
            y = bfr(rng.standard_normal((M, h)).astype(np.float32))
            dev = lambda a: torch.from_numpy(O.to_bf16_bits(a).view(np.int16)).view(torch.bfloat16).cuda()  # noqa
            tok_d, tgt_d = torch.from_numpy(tokens).cuda(), torch.from_numpy(targets).cuda()
            x_d, y_d = torch.empty(M, h, dtype=torch.bfloat16, device="cuda"), dev(y)
            dy_d, loss_d = torch.empty_like(y_d), torch.zeros(1, device="cuda")
            sp = C.c_void_p(s.cuda_stream)
            check(lib().mt_vocab_embed_forward(hv, C.c_void_p(tok_d.data_ptr()), C.c_void_p(x_d.data_ptr()), 0, sp))
            check(lib().mt_vocab_head_loss(hv, C.c_void_p(y_d.data_ptr()), C.c_void_p(tgt_d.data_ptr()),
                                           C.c_void_p(dy_d.data_ptr()), C.c_void_p(loss_d.data_ptr()), sp))
            torch.cuda.synchronize()
            gw = np.empty(vp.value * h, np.float32)
            check(lib().mt_vocab_get_grad(hv, 0, gw.ctypes.data_as(C.POINTER(C.c_float))))
            out.update(x=x_d.float().cpu().numpy(), loss=float(loss_d.item()), dy=dy_d.float().cpu().numpy(),
                       gword=gw.reshape(vp.value, h), v0=v0.value, vp=vp.value,
                       args=(V, h, s_, b, word, pos, g, be, tokens, targets, y))
            lib().mt_vocab_destroy(hv)
        elif mode == "tp_fused":
            # the same TP=2 layer with the forward all-reduces done by NCCL and by the fused
            # GEMM + multimem kernel; with 2 ranks both sum two bf16 values once -> bit-identical
            extra = [Context.unique_id() if rank == 0 else None, Context.unique_id() if rank == 0 else None]
            dist.broadcast_object_list(extra, src=0)
            ids = [obj[0], extra[0], extra[1]]
            d = PL.layer_desc(H, HEADS, S, B, tp_size=world, tp_rank=rank, seed=SEED, layer_index=0)
            params = O.init_params(H, SEED, 0)
            bits = [np.ascontiguousarray(O.to_bf16_bits(p)) for p in params]
            x = O.normal(O.site_seed(SEED, "input", 0, 0), B * S, H)
            g = O.normal(O.site_seed(SEED, "grad", 0, 0), B * S, H, std=1e-2)
            dev = lambda a: torch.from_numpy(O.to_bf16_bits(a).view(np.int16)).view(torch.bfloat16).cuda()  # noqa
            for fused in (0, 1, 2):  # NCCL, fused GEMM + all-reduce, standalone NVLS all-reduce kernel
                os.environ["MT_TP_FUSED"] = "1" if fused == 1 else "0"
                os.environ["MT_TP_NVLS"] = "1" if fused == 2 else "0"
                # the NVLS variant also runs the backward all-reduces through the NVLS kernel
                os.environ["MT_TP_NVLS_BWD"] = "1" if fused == 2 else "0"
                c2 = Context(rank)
                c2.init_comm(ids[fused], world, rank, tensor=world)
                lay = Layer(c2, d)
                for i, b in enumerate(bits):
                    lay.set_param(i, b.ctypes.data)
                xd, gd = dev(x), dev(g)
                yd, dxd = torch.empty_like(xd), torch.empty_like(xd)
                for rep in range(3):  # repeated launches exercise the epoch / counter protocol
                    lay.forward(xd.data_ptr(), yd.data_ptr(), rep, s)
                    lay.backward(gd.data_ptr(), dxd.data_ptr(), rep, s)
                torch.cuda.synchronize()
                out[f"y{fused}"], out[f"dx{fused}"] = yd.float().cpu().numpy(), dxd.float().cpu().numpy()
                lay.close()
                c2.close()
            os.environ.pop("MT_TP_FUSED", None)
            os.environ.pop("MT_TP_NVLS", None)
            os.environ.pop("MT_TP_NVLS_BWD", None)
        elif mode == "peer_hangs":
            # rank 1 builds the same TP=2 stage, then stops taking part (a hung / diverged peer); rank 0's
            # iteration must come back with status 2 within the context's bound (MT_COMM_TIMEOUT_S) —
            # its NCCL all-reduces are released by the host watchdog's ncclCommAbort, the fused
            # GEMM + NVLS reducer (fc2, K = 4h/2 = 4096) by the device-side bounded waits
            import time
            from paper_2201_11990_b200._native import DataError
            ctx.init_comm(obj[0], world, rank, tensor=world, batch=1, micro_batches=1)
            hh = 2048
            st = Stage(ctx, PL.layer_desc(hh, 16, S, B, seed=SEED), 1, 1)
            st.init_params(1, s)
            torch.cuda.synchronize()
            dist.barrier()
            if rank == 1:
                time.sleep(float(os.environ["MT_COMM_TIMEOUT_S"]) * 4 + 20)
                out["status"] = "idle peer"
                q.put((rank, out))
                q.close()
                q.join_thread()  # flush the result before the hard exit
                os._exit(0)  # never touch the communicators again
            xh = torch.zeros(B * S, hh, dtype=torch.bfloat16).pin_memory()
            print("[peer_hangs] rank 0 starts its step alone", flush=True)
            import faulthandler
            faulthandler.dump_traceback_later(90, exit=False)  # where the step blocks, if the bound fails
            t0 = time.monotonic()
            try:
                st.train_step(xh.data_ptr(), xh.data_ptr(), s)
                out["status"] = "completed"
            except DataError as e:
                out["status"], out["msg"] = 2, str(e)
            out["secs"] = time.monotonic() - t0
            print(f"[peer_hangs] rank 0 step returned after {out['secs']:.1f}s: {out['status']}", flush=True)
            out["state"] = ctx.error_state()
            faulthandler.dump_traceback_later(30, exit=False)
            # the GPU must still make progress after the abort (nothing left spinning on it)
            probe = torch.ones(1 << 20, device="cuda")
            out["gpu_alive"] = float((probe * 2).sum().item()) == 2.0 * (1 << 20)
            print("[peer_hangs] gpu alive", out["gpu_alive"], flush=True)
            st.close()
            print("[peer_hangs] stage closed", flush=True)
            ctx.close()
            print("[peer_hangs] context closed", flush=True)
            faulthandler.cancel_dump_traceback_later()
            q.put((rank, out))
            q.close()
            q.join_thread()
            os._exit(0)
        elif mode in ("tp", "tp_sp"):
            ctx.init_comm(obj[0], world, rank, tensor=world)
            sp = mode == "tp_sp"
            if sp:
                ctx.set_sequence_parallel(True)
            d = PL.layer_desc(H, HEADS, S, B, tp_size=world, tp_rank=rank, seed=SEED, layer_index=0)
            lay = Layer(ctx, d)
            params = O.init_params(H, SEED, 0)
            bits = [np.ascontiguousarray(O.to_bf16_bits(p)) for p in params]
            for i, b in enumerate(bits):
                lay.set_param(i, b.ctypes.data)
            x = O.normal(O.site_seed(SEED, "input", 0, 0), B * S, H)
            g = O.normal(O.site_seed(SEED, "grad", 0, 0), B * S, H, std=1e-2)
            dev = lambda a: torch.from_numpy(O.to_bf16_bits(a).view(np.int16)).view(torch.bfloat16).cuda()  # noqa
            rows = slice(rank * (B * S // world), (rank + 1) * (B * S // world)) if sp else slice(None)
            xd, gd = dev(np.ascontiguousarray(x[rows])), dev(np.ascontiguousarray(g[rows]))
            yd, dxd = torch.empty_like(xd), torch.empty_like(xd)
            lay.forward(xd.data_ptr(), yd.data_ptr(), 0, s)
            lay.backward(gd.data_ptr(), dxd.data_ptr(), 0, s)
            if sp:
                lay.finish_grads(s)
            torch.cuda.synchronize()
            out["y"], out["dx"] = yd.float().cpu().numpy(), dxd.float().cpu().numpy()
            grads = []
            for i, p in enumerate(params):
                _, _, (nr, nc) = PL.param_shard(d, i)
                a = np.empty(nr * nc, np.float32)
                lay.get_grad(i, a.ctypes.data)
                grads.append(a.reshape(nr, nc))
            out["grads"] = grads
            lay.close()
        else:
            if mode.startswith("layout"):  # "layout-TP-PP-DP"
                tp, pp, dp = (int(v) for v in mode.split("-")[1:])
                layers, MB = 2 * pp, 4
            else:
                tp, pp, dp = {"pp": (1, world, 1), "dp": (1, 1, world), "tp_stage": (world, 1, 1),
                              "tp_stage_sp": (world, 1, 1)}[mode]
                layers, MB = (2 * pp, 4) if mode == "pp" else (1, 2)
            ctx.init_comm(obj[0], world, rank, tensor=tp, pipeline=pp, data=dp, batch=B * MB * dp, micro_batches=MB)
            place = ctx.placement()
            if mode == "tp_stage_sp":
                ctx.set_sequence_parallel(True)
            d = PL.layer_desc(H, HEADS, S, B, seed=SEED)
            st = Stage(ctx, d, layers, MB)
            per = layers // pp
            for li in range(per):
                params = O.init_params(H, SEED, place.pipeline * per + li)
                for i, p in enumerate(params):
                    b = np.ascontiguousarray(O.to_bf16_bits(p))
                    st.layer(li).set_param(i, b.ctypes.data)
            gids = [place.data * MB + m for m in range(MB)]
            xs = np.stack([O.normal(O.site_seed(SEED, "input", 0, gi), B * S, H) for gi in gids])
            ts = np.stack([O.normal(O.site_seed(SEED, "target", 0, gi), B * S, H) for gi in gids])
            xh = torch.from_numpy(O.to_bf16_bits(xs).view(np.int16)).pin_memory()
            th = torch.from_numpy(O.to_bf16_bits(ts).view(np.int16)).pin_memory()
            for _ in range(2):  # replaying step 0, the second iteration must reproduce the first (grads re-zeroed)
                st.set_step(0)
                loss = st.train_step(xh.data_ptr(), th.data_ptr(), s)
            out["loss"], out["place"] = loss, (place.data, place.pipeline, place.tensor)
            out["h2d"] = st.host_traffic()[0]
            if mode in ("tp_stage", "tp_stage_sp"):  # TP shards: loss + host traffic (grads: test_tensor_parallel_*)
                st.close()
                ctx.close()
                q.put((rank, out))
                return
            from paper_2201_11990_b200.runtime import adam_defaults
            out["grad_norm"] = None
            out["grads"] = []
            dsh = PL.layer_desc(H, HEADS, S, B, tp_size=tp, tp_rank=place.tensor)
            for li in range(per):
                gl = []
                for i in range(len(O.param_shapes(H))):
                    _, _, p = PL.param_shard(dsh, i)
                    a = np.empty(p[0] * p[1], np.float32)
                    st.layer(li).get_grad(i, a.ctypes.data)
                    gl.append(a.reshape(p))
                out["grads"].append(gl)
            # optimizer step: the clip norm is summed over the model-parallel group (PP here)
            out["grad_norm"] = st.optimizer_step(adam_defaults(tokens_seen=2e9, step=1), s)
            st.close()
        ctx.close()
        q.put((rank, out))
    except Exception as e:  # pragma: no cover
        import traceback
        q.put((rank, {"error": traceback.format_exc() + repr(e)}))
    finally:
        try:
            dist.destroy_process_group()
        except Exception:
            pass


def _run(mode, world=2):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    import queue
    import time
    res, deadline = {}, time.monotonic() + 600
    try:
        # a rank that errors (or dies) leaves its peers blocked in NCCL: report it at once instead of
        # waiting out the deadline, and name the ranks that never answered if the deadline passes
        while len(res) < world:
            try:
                r, o = q.get(timeout=5)
            except queue.Empty:
                dead = [i for i, p in enumerate(procs) if p.exitcode not in (None, 0) and i not in res]
                assert not dead, f"{mode}: rank(s) {dead} exited ({[procs[i].exitcode for i in dead]}) without a result"
                assert time.monotonic() < deadline, f"{mode}: no result from rank(s) {sorted(set(range(world)) - set(res))}"
                continue
            res[r] = o
            assert "error" not in o, f"rank {r}: {o['error']}"
    finally:
        for p in procs:
            p.join(timeout=120 if len(res) == world else 1)
            if p.is_alive():
                p.terminate()
    return res


@pytest.mark.timeout(900)
@pytest.mark.parametrize("mode", ["tp", "tp_sp"])
def test_tensor_parallel_layer_two_gpus(mode):
    """TP=2 layer vs the oracle; with sequence parallelism ("tp_sp") each rank holds half of the token
    rows of x / y / dy / dx, and the replicated gradients are completed by finish_grads."""
    _need(2)
    from oracle import oracle as O
    res = _run(mode)
    if mode == "tp_sp":
        for k in ("y", "dx"):
            full = np.concatenate([res[0][k], res[1][k]])
            res[0][k] = res[1][k] = full
    ol = O.OracleLayer(H, HEADS, S, B, 2, dropout_hidden=0.1, dropout_attn=0.1, seed=SEED, layer_index=0,
                       bf16_emulate=True)
    x = O.normal(O.site_seed(SEED, "input", 0, 0), B * S, H)
    g = O.normal(O.site_seed(SEED, "grad", 0, 0), B * S, H, std=1e-2)
    y, dx = ol.forward(x), ol.backward(g)
    for r in (0, 1):
        assert rel(res[r]["y"], y) < 5e-3 and rel(res[r]["dx"], dx) < 1e-2
    from paper_2201_11990_b200 import planner as PL
    for i in range(12):
        full = np.zeros_like(ol.grads[i])
        for r in (0, 1):
            d = PL.layer_desc(H, HEADS, S, B, tp_size=2, tp_rank=r)
            _, (r0, c0), (nr, nc) = PL.param_shard(d, i)
            full[r0:r0 + nr, c0:c0 + nc] = res[r]["grads"][i]
            if nr * nc == H:  # replicated parameter: both ranks hold the full gradient
                assert rel(res[r]["grads"][i], ol.grads[i]) < 1e-2
        assert rel(full, ol.grads[i]) < 1e-2, (i, rel(full, ol.grads[i]))


def _oracle_step(layer_ids, gids):
    from oracle import oracle as O
    ls = [O.OracleLayer(H, HEADS, S, B, 1, dropout_hidden=0.1, dropout_attn=0.1, seed=SEED, layer_index=li,
                        bf16_emulate=True) for li in layer_ids]
    loss = 0.0
    for gi in gids:
        a = O.normal(O.site_seed(SEED, "input", 0, gi), B * S, H)
        for l in ls:
            a = l.forward(a, gi)
        lv, dy = O.mse_loss(a, O.normal(O.site_seed(SEED, "target", 0, gi), B * S, H))
        loss += lv
        for l in reversed(ls):
            dy = l.backward(O.from_bf16_bits(O.to_bf16_bits(dy)), gi)
    return loss, [l.grads for l in ls]


@pytest.mark.timeout(900)
def test_pipeline_parallel_1f1b_two_gpus():
    _need(2)
    res = _run("pp")
    loss, grads = _oracle_step([0, 1, 2, 3], range(4))
    loss, grads = loss / 4, [[g / 4 for g in lg] for lg in grads]  # the batch mean over MB = 4
    assert abs(res[1]["loss"] - loss) / loss < 5e-3, (res[1]["loss"], loss)
    norm = np.sqrt(sum(float((g.astype(np.float64) ** 2).sum()) for lg in grads for g in lg))
    for r in (0, 1):
        assert abs(res[r]["grad_norm"] - norm) / norm < 2e-2, (res[r]["grad_norm"], norm)
    for r in (0, 1):
        for li in range(2):
            for i in range(12):
                assert rel(res[r]["grads"][li][i], grads[2 * r + li][i]) < 2e-2, (r, li, i)


@pytest.mark.timeout(900)
def test_data_parallel_gradient_allreduce_two_gpus():
    _need(2)
    res = _run("dp")
    loss, grads = _oracle_step([0], range(4))  # DP = 2 replicas x MB = 2: the mean over all 4 microbatches
    for r in (0, 1):
        assert abs(res[r]["loss"] - loss / 4) / loss < 5e-3
        norm = np.sqrt(sum(float(((g / 4).astype(np.float64) ** 2).sum()) for g in grads[0]))
        assert abs(res[r]["grad_norm"] - norm) / norm < 2e-2
        for i in range(12):
            assert rel(res[r]["grads"][0][i], grads[0][i] / 4) < 2e-2, (r, i)


@pytest.mark.timeout(900)
def test_vocab_parallel_head_two_gpus():
    """N3 at TP=2: each rank holds half of the (padded) vocabulary; the loss, the embedding output
    and dL/dy agree with the unsharded numpy reference on both ranks; the word-embedding gradient
    shards tile the full gradient."""
    _need(2)
    from tests.test_vocab_gpu import reference
    res = _run("vocab")
    V, h, s_, b, word, pos, g, be, tokens, targets, y = res[0]["args"]
    x_ref, loss_ref, dy_ref, dword_ref, _, _, _ = reference(V, h, s_, b, 0.1, word, pos, g, be, tokens, targets, y,
                                                            np.zeros((s_ * b, h), np.float32))
    full = np.zeros_like(dword_ref)
    for r in (0, 1):
        assert rel(res[r]["x"], x_ref) < 5e-3
        assert abs(res[r]["loss"] - loss_ref) / loss_ref < 2e-3
        assert rel(res[r]["dy"], dy_ref) < 2e-2
        full[res[r]["v0"]:res[r]["v0"] + res[r]["vp"]] = res[r]["gword"]
    assert rel(full, dword_ref) < 2e-2


@pytest.mark.timeout(900)
def test_language_model_pipeline_two_gpus():
    """Token ids -> embedding (stage 0) -> 1F1B over PP=2 -> tied head + cross-entropy (stage 1):
    loss, every layer gradient, the tied word-embedding gradient (all-reduced between the first and
    the last stage), the position / final-LN gradients and the clipped-norm all equal the same model
    run unpartitioned (PP = 1) on one GPU (1e-5 relative: only float summation order differs)."""
    _need(2)
    res = _run("lm_pp")
    ref = res[0]["ref"]
    assert abs(res[1]["pp"]["loss"] - ref["loss"]) <= 1e-5 * ref["loss"], (res[1]["pp"]["loss"], ref["loss"])
    assert res[0]["pp"]["loss"] == 0.0
    for r in (0, 1):
        assert abs(res[r]["ref"]["loss"] - ref["loss"]) <= 1e-6 * ref["loss"]
        for p in range(12):
            assert rel(res[r]["pp"]["layers"][0][p], ref["layers"][r][p]) < 1e-5, (r, p)
        assert rel(res[r]["pp"]["vocab"][0], ref["vocab"][0]) < 1e-5, r  # tied E: both ends hold the sum
        assert abs(res[r]["pp"]["norm"] - ref["norm"]) <= 1e-4 * ref["norm"], (res[r]["pp"]["norm"], ref["norm"])
    assert rel(res[0]["pp"]["vocab"][1], ref["vocab"][1]) < 1e-5  # position embedding: first stage
    for p in (2, 3):  # final LayerNorm: last stage
        assert rel(res[1]["pp"]["vocab"][p], ref["vocab"][p]) < 1e-5


@pytest.mark.timeout(900)
@pytest.mark.parametrize("mode", ["tp_stage", "tp_stage_sp"])
def test_tensor_parallel_stage_host_inputs_two_gpus(mode):
    """Stage at TP=2 fed from host buffers: each TP rank copies half of every input / target over
    PCIe (all-gathered over NVLink, or kept as the rank's rows under sequence parallelism); the loss
    equals the oracle's."""
    _need(2)
    res = _run(mode)
    loss, _ = _oracle_step([0], range(2))
    loss /= 2  # the batch mean over MB = 2
    full = 2 * 2 * (B * S * H * 2)  # MB=2 inputs + targets, bf16
    for r in (0, 1):
        assert abs(res[r]["loss"] - loss) / loss < 5e-3, (res[r]["loss"], loss)
        assert res[r]["h2d"] == full // 2, res[r]["h2d"]


@pytest.mark.timeout(600)
def test_fused_gemm_allreduce_matches_nccl_two_gpus():
    """Forward row-parallel GEMM + TP all-reduce fused in one kernel (a reducer kernel reduces finished
    tiles over NVLink SHARP with multimem.ld_reduce / multimem.st) at TP=2 over repeated launches:
    within the oracle tolerance of test_tensor_parallel_layer_two_gpus, within bf16 noise of the
    GEMM + ncclAllReduce path (the two sums differ by one bf16 ulp on rare elements, which the later
    GEMMs spread; measured unbiased), and the TP replicas of the fused result are bit-identical (one
    owner computes each unit and multicasts it). The standalone-NVLS variant also runs the two backward
    LN-input-gradient all-reduces through the NVLS kernel on the side stream (MT_TP_NVLS_BWD=1)."""
    _need(2)
    from oracle import oracle as O
    res = _run("tp_fused")
    ol = O.OracleLayer(H, HEADS, S, B, 2, dropout_hidden=0.1, dropout_attn=0.1, seed=SEED, layer_index=0,
                       bf16_emulate=True)
    x = O.normal(O.site_seed(SEED, "input", 0, 0), B * S, H)
    g = O.normal(O.site_seed(SEED, "grad", 0, 0), B * S, H, std=1e-2)
    y, dx = ol.forward(x, 2), ol.backward(g, 2)  # the worker's last repetition is microbatch 2
    for r in (0, 1):
        assert rel(res[r]["y0"], y) < 5e-3
        for v in ("1", "2"):  # fused GEMM + all-reduce; standalone NVLS all-reduce kernel
            assert rel(res[r]["y" + v], y) < 5e-3 and rel(res[r]["dx" + v], dx) < 1e-2
            assert rel(res[r]["y" + v], res[r]["y0"]) < 5e-3 and rel(res[r]["dx" + v], res[r]["dx0"]) < 5e-3
    for v in ("1", "2"):
        assert np.array_equal(res[0]["y" + v], res[1]["y" + v])
        assert np.array_equal(res[0]["dx" + v], res[1]["dx" + v])


@pytest.mark.timeout(900)
def test_tensor_parallel_layer_four_gpus():
    """TP=4 layer (the NVLink SHARP all-reduce kernel is the default forward all-reduce from TP=4)
    against the oracle: every rank's replicated output and input gradient."""
    _need(4)
    from oracle import oracle as O
    res = _run("tp", world=4)
    ol = O.OracleLayer(H, HEADS, S, B, 4, dropout_hidden=0.1, dropout_attn=0.1, seed=SEED, layer_index=0,
                       bf16_emulate=True)
    x = O.normal(O.site_seed(SEED, "input", 0, 0), B * S, H)
    g = O.normal(O.site_seed(SEED, "grad", 0, 0), B * S, H, std=1e-2)
    y, dx = ol.forward(x), ol.backward(g)
    for r in range(4):
        assert rel(res[r]["y"], y) < 5e-3 and rel(res[r]["dx"], dx) < 1e-2, r
    assert all(np.array_equal(res[0]["y"], res[r]["y"]) for r in range(1, 4))


@pytest.mark.timeout(900)
@pytest.mark.parametrize("layout", [(2, 2, 1), (2, 1, 2), (1, 2, 2)], ids=["tp2pp2", "tp2dp2", "pp2dp2"])
def test_two_axis_layouts_four_gpus(layout):
    """Every two-axis composition of the 3D layout on 4 GPUs (TPxPP, TPxDP, PPxDP; 2 layers per stage,
    MB=4 per replica): the rank placement is curator::map_topology's (pp slowest, tp fastest), the loss
    is the mean over all DP x MB microbatches of the oracle's losses, every rank's gradient shard equals
    the matching slice of the oracle's gradients over the same mean, and the clip norm is the global one."""
    _need(4)
    tp, pp, dp = layout
    from paper_2201_11990_b200 import planner as PL
    res = _run(f"layout-{tp}-{pp}-{dp}", world=4)
    MB = 4
    for r in range(4):  # rank = (pp * DP + dp) * TP + tp  (planner.cpp:110-126)
        dpi, ppi, tpi = res[r]["place"]
        assert r == (ppi * dp + dpi) * tp + tpi, (r, res[r]["place"])
    loss, grads = _oracle_step(list(range(2 * pp)), range(dp * MB))
    loss, grads = loss / MB, [[g / MB for g in lg] for lg in grads]  # per-replica batch mean
    norm = np.sqrt(sum(float(((g / dp).astype(np.float64) ** 2).sum()) for lg in grads for g in lg))
    for r in range(4):
        dpi, ppi, tpi = res[r]["place"]
        if ppi == pp - 1:
            assert abs(res[r]["loss"] - loss / dp) / loss < 5e-3, (r, res[r]["loss"], loss / dp)
        assert abs(res[r]["grad_norm"] - norm) / norm < 2e-2, (r, res[r]["grad_norm"], norm)
        d = PL.layer_desc(H, HEADS, S, B, tp_size=tp, tp_rank=tpi)
        for li in range(2):
            for i in range(12):
                _, (r0, c0), (nr, nc) = PL.param_shard(d, i)
                ref = grads[2 * ppi + li][i][r0:r0 + nr, c0:c0 + nc] / dp
                assert rel(res[r]["grads"][li][i], ref) < 2e-2, (r, li, i, rel(res[r]["grads"][li][i], ref))
    # DP replicas hold bit-identical gradients after the all-reduce
    for r in range(4):
        for q in range(r + 1, 4):
            if res[r]["place"][1:] == res[q]["place"][1:]:
                for li in range(2):
                    for i in range(12):
                        assert np.array_equal(res[r]["grads"][li][i], res[q]["grads"][li][i]), (r, q, li, i)


@pytest.mark.timeout(240)
def test_hung_peer_surfaces_as_status_2(monkeypatch):
    """a peer that stops participating must not wedge the GPU. With a 10 s bound, rank
    0's training step returns status 2 (DataError) within the bound (+ drain), and the context reports
    its communicators aborted."""
    _need(2)
    monkeypatch.setenv("MT_COMM_TIMEOUT_S", "10")
    res = _run("peer_hangs")
    r0 = res[0]
    assert r0["status"] == 2, r0
    assert r0["secs"] < 10 + 5 + 60, r0
    assert r0["state"] == 3 and r0["gpu_alive"], r0
    assert "aborted" in r0["msg"], r0
