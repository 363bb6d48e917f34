"""1F1B schedule, shard layout and seeded streams (no GPU). Bit-exact: op lists, shard ranges.

The reference gives only the bubble formula (proj/src/planner.cpp:27-32); the
schedule is pinned to it: a dependency-respecting simulation of one_f_one_b with integer op costs
has makespan (MB + PP - 1)(tF + tB) exactly, i.e. efficiency == curator::pipeline_efficiency.
"""
import pytest

from paper_2201_11990_b200 import planner as PL


def test_one_f_one_b_golden_pp4_mb16_stage0():
    ops = PL.pipeline_schedule(0, 4, 16)
    want = [("F", 0), ("F", 1), ("F", 2), ("F", 3), ("B", 0)]
    for i in range(4, 16):
        want += [("F", i), ("B", i - 3)]
    want += [("B", 13), ("B", 14), ("B", 15)]
    assert ops == want


@pytest.mark.parametrize("pp", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("mb", [1, 2, 3, 4, 8, 16, 32])
def test_schedule_shape(pp, mb):
    for stage in range(pp):
        ops = PL.pipeline_schedule(stage, pp, mb)
        assert len(ops) == 2 * mb
        assert [m for k, m in ops if k == "F"] == list(range(mb))
        assert [m for k, m in ops if k == "B"] == list(range(mb))
        warm = min(pp - stage - 1, mb)
        assert all(k == "F" for k, _ in ops[:warm])
        # in flight never exceeds warmup + 1 (the 1F1B memory bound)
        inflight = peak = 0
        for k, _ in ops:
            inflight += 1 if k == "F" else -1
            peak = max(peak, inflight)
        assert peak == min(warm + 1, mb)


@pytest.mark.parametrize("pp", range(1, 9))
@pytest.mark.parametrize("mb", [1, 2, 3, 5, 8, 16, 32])
@pytest.mark.parametrize("tf,tb", [(1, 1), (1, 2), (2, 3)])
def test_simulated_bubble_equals_planner_formula(pp, mb, tf, tb):
    makespan = PL.pipeline_simulate(pp, mb, tf, tb)
    assert makespan == (mb + pp - 1) * (tf + tb)
    assert mb * (tf + tb) / makespan == pytest.approx(PL.pipeline_efficiency(mb, pp), rel=1e-15)


def test_schedule_errors():
    with pytest.raises(PL.ConfigError):
        PL.pipeline_schedule(4, 4, 8)
    with pytest.raises(PL.ConfigError):
        PL.pipeline_schedule(0, 0, 8)


@pytest.mark.parametrize("h,H,t", [(256, 4, 2), (12288, 96, 8), (20480, 128, 8), (8192, 64, 2)])
def test_tensor_shards_tile_the_global_parameters(h, H, t):
    hd = h // H
    seen = {}
    for r in range(t):
        d = PL.layer_desc(h, H, 2048, 1, tp_size=t, tp_rank=r)
        for p in range(12):
            (gr, gc), (r0, c0), (nr, nc) = PL.param_shard(d, p)
            seen.setdefault(p, []).append((r0, c0, nr, nc, gr, gc))
    for p, blocks in seen.items():
        gr, gc = blocks[0][4], blocks[0][5]
        if gr * gc in (h,):  # replicated vectors (LN params, row-parallel biases)
            assert all(b[:4] == (0, 0, 1, h) for b in blocks)
            continue
        area = sum(b[2] * b[3] for b in blocks)
        assert area == gr * gc, (p, blocks)
    # QKV rows of rank r = heads [r*H/t, (r+1)*H/t) in (head, {q,k,v}, hd) order
    d = PL.layer_desc(h, H, 2048, 1, tp_size=t, tp_rank=t - 1)
    _, (r0, _), (nr, _) = PL.param_shard(d, 2)
    assert r0 == (t - 1) * (H // t) * 3 * hd and nr == (H // t) * 3 * hd


def test_shard_errors():
    with pytest.raises(PL.ConfigError):
        PL.param_shard(PL.layer_desc(256, 4, 128, 1, tp_size=8, tp_rank=0), 2)  # 4 heads over 8 ranks


def test_stream_keys_follow_reference_seed_pattern():
    # mix64(seed, fnv1a64(name) ^ (layer << 32 | mb)), reference hashing.hpp:13-63 / pipeline.cpp:708-711
    M = (1 << 64) - 1

    def splitmix(z):
        z = (z + 0x9E3779B97F4A7C15) & M
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        return z ^ (z >> 31)

    def fnv(s):
        h = 0xCBF29CE484222325
        for c in s.encode():
            h = ((h ^ c) * 0x100000001B3) & M
        return h

    for name, layer, mb in (("attn.probs", 0, 0), ("qkv.weight", 7, 0), ("input", 0, 15)):
        want = splitmix(20260808 ^ splitmix(fnv(name) ^ ((layer << 32) | mb)))
        assert PL.stream_key(20260808, name, layer, mb) == want
    assert PL.dropout_threshold16(0.1) == round(0.1 * 65536)
    assert PL.dropout_threshold16(0.0) == 0
