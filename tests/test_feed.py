"""Blend-driven data feed, CPU only.

* curator::next_batch_composition: the reference's own unit tests (proj/tests/unit/test_blending.cpp)
  compiled unmodified against our blending.cpp, and a live bit-exact diff of the count and credit
  streams against the reference's blending.cpp (oracle/_ref/libcurator_ref.so) over random mixes.
* mt_blend_manifest: byte-identical to blend_manifest.jsonl files written by the reference pipeline
  itself (tests/golden/blend, recorded by tests/golden/make_blend_golden.py).
* mt_feed: manifest -> global batch -> DP slice -> microbatches, token windows, error behaviour.
"""
import ctypes as C
import json
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_2201_11990_b200._native import ConfigError, DataError
from paper_2201_11990_b200.feed import Blend, Feed, blend_manifest, doc_tokens
from paper_2201_11990_b200.planner import batch_size_at

ROOT = Path(__file__).resolve().parents[1]
GOLD = ROOT / "tests" / "golden" / "blend"
REF_SO = ROOT / "oracle" / "_ref" / "libcurator_ref.so"


@pytest.mark.skipif(not (ROOT / "oracle" / "_ref" / "test_blending_mine").exists(), reason="reference not built")
def test_reference_blending_unit_tests_pass_unmodified_against_ours():
    for exe in ("test_blending_mine", "test_blending_ref"):
        r = subprocess.run([str(ROOT / "oracle" / "_ref" / exe)], capture_output=True, text=True)
        assert r.returncode == 0, r.stdout + r.stderr
        assert "8 passed | 0 failed" in r.stdout, r.stdout


FIFTEEN = [14.3, 19.3, 5.7, 2.9, 4.8, 0.9, 1.0, 0.2, 1.4, 1.6, 9.4, 13.0, 15.7, 9.0, 0.9]  # test_blending.cpp:15-24


@pytest.mark.skipif(not REF_SO.exists(), reason="reference not built")
@pytest.mark.parametrize("case", range(12))
def test_blend_stream_bit_exact_vs_reference(case):
    ref = C.CDLL(str(REF_SO))
    rng = np.random.default_rng(case)
    if case == 0:
        w, batch = np.array(FIFTEEN), 1920
    elif case == 1:
        w, batch = np.array([1 / 3, 1 / 3, 1 - 2 / 3]), 7
    else:
        n = int(rng.integers(1, 16))
        w = rng.random(n) ** 3 + 1e-3
        batch = int(rng.integers(1, 2500))
    steps, n = 400, len(w)
    counts = np.empty(steps * n, np.uint64)
    credit = np.empty(steps * n, np.float64)
    ww = np.ascontiguousarray(w, np.float64)
    ref.ref_blend_run.argtypes = [C.c_int32, C.c_void_p, C.c_int32, C.c_uint64, C.c_int64, C.c_void_p, C.c_void_p]
    assert ref.ref_blend_run(n, ww.ctypes.data, 1, batch, steps, counts.ctypes.data, credit.ctypes.data) == 0
    b = Blend([f"d{i}" for i in range(n)], w, normalize=True)
    for t in range(steps):
        c, cr, d = b.next(batch)
        assert np.array_equal(c, counts[t * n:(t + 1) * n]), t
        assert np.array_equal(cr.view(np.uint64), credit[t * n:(t + 1) * n].view(np.uint64)), t  # bitwise
        assert int(c.sum()) == batch
        assert np.all(np.abs(cr) < 1.0)
    b.close()


def test_blend_errors_and_ties():
    with pytest.raises(ConfigError, match="sum to"):
        Blend(["a", "b"], [0.5, 0.6])
    with pytest.raises(ConfigError, match="weight must be in"):
        Blend(["a", "b"], [0.0, 1.0])
    b = Blend(["a", "b", "c", "d"], [0.25] * 4)
    assert b.next(2)[0].tolist() == [1, 1, 0, 0]  # remainder ties: dataset order
    assert b.next(2)[0].tolist() == [0, 0, 1, 1]
    with pytest.raises(ConfigError):
        b.next(0)
    b.close()


CASES = json.loads((GOLD / "cases.json").read_text(encoding="utf-8"))


@pytest.mark.parametrize("case", sorted(CASES))
def test_blend_manifest_byte_identical_to_reference_pipeline(case, tmp_path):
    c = CASES[case]
    out = tmp_path / "blend_manifest.jsonl"
    blend_manifest(out, [(d["name"], d["weight"], d["doc_ids"]) for d in c["datasets"]], c["steps"],
                   c["batch_size"], shuffle=c["shuffle"], config_seed=c["seed"])
    assert out.read_bytes() == (GOLD / f"{case}.jsonl").read_bytes()


def test_blend_manifest_no_documents_and_errors(tmp_path):
    out = tmp_path / "m.jsonl"
    blend_manifest(out, [("a", 1.0, [])], 3, 4)  # nothing available: zero steps drawn, empty manifest
    assert out.read_bytes() == b""
    with pytest.raises(DataError, match="positive weight but no documents"):
        blend_manifest(out, [("a", 0.5, [1, 2]), ("b", 0.5, [])], 3, 4)
    with pytest.raises(ConfigError, match="steps >= 1"):
        blend_manifest(out, [("a", 1.0, [1])], 0, 4)


def _lines(path):
    return [json.loads(x) for x in Path(path).read_text(encoding="utf-8").splitlines()]


@pytest.mark.parametrize("dp", [1, 2, 4])
def test_feed_splits_global_batch_into_dp_slices_and_microbatches(dp):
    path = GOLD / "percent_mix.jsonl"  # 20 steps x 32 samples
    rows = _lines(path)
    V, s, b = 1000, 16, 2
    feeds = [Feed(path, V, s, b, dp, r, seed=99) for r in range(dp)]
    assert feeds[0].steps() == 20
    for step in (0, 7, 19):
        G, MB = feeds[0].step_info(step)
        assert G == 32 and MB == 32 // (b * dp)
        batch = [r for r in rows if r["step"] == step]
        for r, f in enumerate(feeds):
            tok = np.zeros((MB, b * s), np.int32)
            tgt = np.zeros((MB, b * s), np.int32)
            f.fill(step, tok, tgt, MB)
            for j in range(G // dp):  # sample j of rank r = manifest sample r*G/dp + j
                want = batch[r * (G // dp) + j]
                ds, doc = f.sample(step, r * (G // dp) + j)
                assert (f.dataset_name(ds), doc) == (want["dataset"], want["doc_id"])
                stream = doc_tokens(99, want["dataset"], want["doc_id"], V, s + 1)
                m, row = divmod(j, b)
                assert np.array_equal(tok[m, row * s:(row + 1) * s], stream[:s])
                assert np.array_equal(tgt[m, row * s:(row + 1) * s], stream[1:])
    for f in feeds:
        f.close()


def test_feed_token_stream_properties():
    a = doc_tokens(1, "web", 5, 50257, 4096)
    assert a.min() >= 0 and a.max() < 50257
    assert np.array_equal(a, doc_tokens(1, "web", 5, 50257, 4096))
    assert not np.array_equal(a, doc_tokens(2, "web", 5, 50257, 4096))
    assert not np.array_equal(a, doc_tokens(1, "books", 5, 50257, 4096))
    assert len(np.unique(a)) > 3900  # no short cycle


def test_feed_batch_ramp_and_errors(tmp_path):
    # global batch from the reference's ramp (batch_size_at: 32 -> 1920 in steps of 32), scaled by 1/8
    ramp = [batch_size_at(t * 2e8) // 8 for t in range(6)]
    assert ramp[0] == 4 and ramp == sorted(ramp)
    m = tmp_path / "ramp.jsonl"
    blend_manifest(m, [("a", 0.7, list(range(100))), ("b", 0.3, list(range(1000, 1050)))], 6, 0,
                   batch_per_step=ramp)
    f = Feed(m, 512, 8, 2, 2, 1)
    assert [f.step_info(t)[0] for t in range(6)] == ramp
    assert [f.step_info(t)[1] for t in range(6)] == [g // 4 for g in ramp]
    with pytest.raises(ConfigError, match="buffers hold"):
        f.fill(5, np.zeros(ramp[5] * 8, np.int32), None, 1)
    f.close()
    f = Feed(m, 512, 8, 3, 1, 0)  # 4 samples are not a multiple of micro_batch 3
    with pytest.raises(ConfigError, match="not a multiple"):
        f.step_info(0)
    f.close()
    bad = tmp_path / "bad.jsonl"
    bad.write_text('{"step":0,"dataset":"a","doc_id":1}\n{"step":0,"dataset":"a"}\n')
    with pytest.raises(DataError, match="line 2"):
        Feed(bad, 512, 8, 1)
    bad.write_text('{"step":1,"dataset":"a","doc_id":1}\n{"step":0,"dataset":"a","doc_id":2}\n')
    with pytest.raises(DataError, match="non-decreasing"):
        Feed(bad, 512, 8, 1)
    with pytest.raises(DataError, match="cannot open"):
        Feed(tmp_path / "missing.jsonl", 512, 8, 1)
    with pytest.raises(ConfigError):
        Feed(m, 512, 8, 1, 2, 2)  # dp_rank out of range
