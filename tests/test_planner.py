"""curator:: planner parity (no GPU): libmtnlg.so's C ABI against the reference planner.

* golden vectors recorded from the reference's own planner (tests/golden/planner_golden.json, made
  by tests/golden/make_planner_golden.py from /root/reference/proj/src/planner.cpp) — bit-exact;
* the reference's unit tests (proj/tests/unit/test_planner.cpp, 16 cases) compiled UNMODIFIED
  against this framework's planner through oracle/doctest_shim (only where /root/reference exists);
* a live differential sweep against oracle/_ref/libcurator_ref.so when it is built.
"""
import ctypes as C
import json
import os
import subprocess
import tempfile
from pathlib import Path

import pytest

from paper_2201_11990_b200 import planner as PL
from paper_2201_11990_b200._native import ModelShape, ParallelConfig, lib

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = json.loads((ROOT / "tests" / "golden" / "planner_golden.json").read_text())


def _ours_f64(fn, *args):
    out = C.c_double()
    rc = fn(*args, C.byref(out))
    return {"error": rc, "message": lib().mt_last_error().decode()} if rc else out.value.hex()


def test_map_topology_golden():
    for case in GOLDEN["map_topology"]:
        nodes, gpn, tp, pp, dp = case["args"]
        want = case["out"]
        if "error" in want:
            with pytest.raises(PL.ConfigError) as ei:
                PL.map_topology(PL.topology(nodes, gpn), PL.parallel(tp, pp, dp))
            assert str(ei.value) == want["message"]
        else:
            got = PL.map_topology(PL.topology(nodes, gpn), PL.parallel(tp, pp, dp))
            assert [[p.data, p.pipeline, p.tensor, p.node, p.gpu] for p in got] == want["ranks"], case["args"]


def test_scalar_formulas_golden():
    L = lib()
    for c in GOLDEN["pipeline_efficiency"]:
        assert _ours_f64(L.mt_pipeline_efficiency, *c["args"]) == c["out"], c
    for c in GOLDEN["lr_at"]:
        assert _ours_f64(L.mt_lr_at, float.fromhex(c["args"][0])) == c["out"], c
    for c in GOLDEN["weight_init_std"]:
        assert _ours_f64(L.mt_weight_init_std, float.fromhex(c["args"][0])) == c["out"], c
    for c in GOLDEN["activation_bytes"]:
        assert _ours_f64(L.mt_activation_bytes, *map(float, c["args"])) == c["out"], c
    for c in GOLDEN["model_state_bytes"]:
        assert _ours_f64(L.mt_model_state_bytes, float.fromhex(c["args"][0])) == c["out"], c
    for c in GOLDEN["batch_size_at"]:
        out = C.c_int32()
        rc = L.mt_batch_size_at(float.fromhex(c["args"][0]), C.byref(out))
        assert (out.value if rc == 0 else {"error": rc}) == c["out"], c
    for c in GOLDEN["estimated_tflops_per_gpu"]:
        P, Ly, h, H, s, nodes, gpn, B, secs = c["args"]
        sh = ModelShape(P, Ly, h, H, s, 50257)
        t, par = PL.topology(nodes, gpn), ParallelConfig(1, 1, 1, B, 1)
        got = _ours_f64(L.mt_estimated_tflops_per_gpu, C.byref(sh), C.byref(par), C.byref(t), float.fromhex(secs))
        assert got == c["out"], c


def test_plan_report_golden():
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "plan.txt")
        for c in GOLDEN["plan_report"]:
            Path(path).write_text(c["config"])
            for key, as_json in (("text", False), ("json", True)):
                want = c[key]
                if isinstance(want, dict):
                    with pytest.raises(PL.ConfigError) as ei:
                        PL.plan_report(path, as_json)
                    assert str(ei.value).replace(d, "<dir>") == want["message"], c["name"]
                elif as_json:
                    assert json.loads(PL.plan_report(path, True)) == json.loads(want), c["name"]
                else:
                    assert PL.plan_report(path, False) == want, c["name"]
    with pytest.raises(PL.ConfigError):
        PL.plan_report("/nonexistent/plan.txt")


def test_paper_operating_points():
    # PAPER.md:188-192 and :271 via the reference's formulas
    assert PL.pipeline_efficiency(140, 35) == 140.0 / 174.0
    assert PL.pipeline_efficiency(280, 35) == 280.0 / 314.0
    assert PL.model_state_bytes(530e9) == 1.06e13
    assert PL.batch_size_at(6e9) == 992


REF_TREE = Path("/root/reference/proj/tests/unit/test_planner.cpp")


@pytest.mark.skipif(not REF_TREE.exists(), reason="reference tree not mounted (GPU box)")
def test_reference_unit_tests_pass_unmodified_against_our_planner():
    subprocess.run(["make", "-s", "-C", str(ROOT / "oracle"), "ref"], check=True)
    for exe in ("test_planner_mine", "test_planner_ref"):
        r = subprocess.run([str(ROOT / "oracle" / "_ref" / exe)], capture_output=True, text=True)
        assert r.returncode == 0, r.stdout + r.stderr
        assert "16 passed | 0 failed" in r.stdout, r.stdout


@pytest.mark.skipif(not (ROOT / "oracle" / "_ref" / "libcurator_ref.so").exists(), reason="reference not built")
def test_live_differential_sweep():
    ref = C.CDLL(str(ROOT / "oracle" / "_ref" / "libcurator_ref.so"))
    ref.ref_pipeline_efficiency.argtypes = [C.c_int32, C.c_int32, C.POINTER(C.c_double)]
    ref.ref_lr_at.argtypes = [C.c_double, C.POINTER(C.c_double)]
    ref.ref_batch_size_at.argtypes = [C.c_double, C.POINTER(C.c_int32)]
    for mb in range(1, 65):
        for pp in range(1, 40):
            a, b = C.c_double(), C.c_double()
            ref.ref_pipeline_efficiency(mb, pp, C.byref(a))
            lib().mt_pipeline_efficiency(mb, pp, C.byref(b))
            assert a.value == b.value
    for i in range(2000):
        t = i * 2.3e8
        a, b = C.c_double(), C.c_double()
        ref.ref_lr_at(t, C.byref(a))
        lib().mt_lr_at(t, C.byref(b))
        assert a.value == b.value
        x, y = C.c_int32(), C.c_int32()
        ref.ref_batch_size_at(t / 30, C.byref(x))
        lib().mt_batch_size_at(t / 30, C.byref(y))
        assert x.value == y.value
