"""Multi-process (world_size 2, gloo, CPU) coverage of the N>1 host logic:

* TP=2: each rank derives its groups from curator::map_topology and its weight shards from
  mt_param_shard, computes its row-parallel partial of the MLP block, all-reduces over its TP
  group and matches the unsharded result (the Megatron f/g structure the GPU runtime uses);
* PP=2 with 1F1B: two processes each own one oracle layer, run mt_pipeline_schedule's op order with
  activations / gradients exchanged point-to-point (paired like the runtime's NCCL groups) and
  reproduce the single-process two-layer result (loss, dx, every parameter gradient).
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2201_11990_b200 import planner as PL  # noqa: E402

SEED = 20260808


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _tp_worker(rank, world, port, q):
    try:
        _init(rank, world, port)
        h, H, M = 64, 4, 32
        place = PL.map_topology(PL.topology(1, world), PL.parallel(tensor=world))[rank]
        assert place.tensor == rank and place.pipeline == 0 and place.data == 0
        params = O.init_params(h, SEED, 0)
        d = PL.layer_desc(h, H, 32, 1, tp_size=world, tp_rank=place.tensor)
        (_, _), (r0, _), (nr, _) = PL.param_shard(d, 8)     # fc1.weight rows
        (_, _), (_, c0), (_, nc) = PL.param_shard(d, 10)    # fc2.weight cols
        x = O.normal(O.site_seed(SEED, "input", 0, 0), M, h)
        w1, w2 = params[8], params[10]
        a = np.maximum(x @ w1[r0:r0 + nr].T, 0)             # column-parallel (no comm)
        part = torch.from_numpy(a @ w2[:, c0:c0 + nc].T)    # row-parallel partial
        dist.all_reduce(part)                               # "g"
        full = np.maximum(x @ w1.T, 0) @ w2.T
        q.put((rank, float(np.abs(part.numpy() - full).max())))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def _pp_worker(rank, world, port, q):
    try:
        _init(rank, world, port)
        h, H, s, MB = 64, 4, 32, 4
        place = PL.map_topology(PL.topology(1, world), PL.parallel(pipeline=world, micro_batches=MB))[rank]
        stage = place.pipeline
        (lo, hi) = (stage, stage + 1)  # one layer per stage
        layer = O.OracleLayer(h, H, s, 1, 1, dropout_hidden=0.1, dropout_attn=0.1, seed=SEED, layer_index=lo,
                              bf16_emulate=False)
        ops = PL.pipeline_schedule(stage, world, MB)
        loss = 0.0
        pending = []  # sends are posted asynchronously (the runtime pairs them in NCCL groups)
        for kind, mb in ops:
            if kind == "F":
                if stage == 0:
                    x = O.normal(O.site_seed(SEED, "input", 0, mb), s, h)
                else:
                    t = torch.empty(s, h)
                    dist.recv(t, stage - 1)
                    x = t.numpy()
                y = layer.forward(x, mb)
                if stage == world - 1:
                    tgt = O.normal(O.site_seed(SEED, "target", 0, mb), s, h)
                    l, dy = O.mse_loss(y, tgt)
                    loss += l
                    dx = layer.backward(dy, mb)  # last stage: 1F1B runs B(mb) right after F(mb)
                    pending.append(dist.isend(torch.from_numpy(dx), stage - 1))
                else:
                    pending.append(dist.isend(torch.from_numpy(y), stage + 1))
            elif stage != world - 1:
                g = torch.empty(s, h)
                dist.recv(g, stage + 1)
                layer.backward(g.numpy(), mb)
        for w in pending:
            w.wait()
        q.put((rank, loss, [gr.copy() for gr in layer.grads]))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e), None))
    finally:
        dist.destroy_process_group()


def _run(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=fn, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    return sorted(out, key=lambda t: t[0])


@pytest.mark.timeout(300)
def test_tensor_parallel_allreduce_over_gloo():
    for rank, err in _run(_tp_worker):
        assert isinstance(err, float) and err < 1e-4, (rank, err)


@pytest.mark.timeout(300)
def test_one_f_one_b_pipeline_over_gloo_matches_single_process():
    res = _run(_pp_worker)
    assert all(r[2] is not None for r in res), res
    h, H, s, MB = 64, 4, 32, 4
    l0 = O.OracleLayer(h, H, s, 1, 1, dropout_hidden=0.1, dropout_attn=0.1, seed=SEED, layer_index=0,
                       bf16_emulate=False)
    l1 = O.OracleLayer(h, H, s, 1, 1, dropout_hidden=0.1, dropout_attn=0.1, seed=SEED, layer_index=1,
                       bf16_emulate=False)
    loss = 0.0
    for mb in range(MB):
        x = O.normal(O.site_seed(SEED, "input", 0, mb), s, h)
        y = l1.forward(l0.forward(x, mb), mb)
        l, dy = O.mse_loss(y, O.normal(O.site_seed(SEED, "target", 0, mb), s, h))
        loss += l
        l0.backward(l1.backward(dy, mb), mb)
    assert res[1][1] == pytest.approx(loss, rel=1e-6)
    for got, want in ((res[0][2], l0.grads), (res[1][2], l1.grads)):
        for a, b in zip(got, want):
            np.testing.assert_allclose(a, b, rtol=1e-5, atol=1e-8)
