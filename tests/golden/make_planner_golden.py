"""Generate tests/golden/planner_golden.json from the REFERENCE planner (test infrastructure).

Runs in the build container only: it loads oracle/_ref/libcurator_ref.so, i.e. the reference's own
proj/src/planner.cpp compiled unmodified by oracle/Makefile, and records its outputs (doubles as
float.hex, so comparisons are bit-exact) for the planner functions on the hot path
 over grids covering the five BASELINE.json layouts, the paper's
operating points and the error paths. tests/test_planner.py checks libmtnlg.so against this file.

    python tests/golden/make_planner_golden.py
"""
import ctypes as C
import json
import os
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from paper_2201_11990_b200._native import ClusterTopology, ModelShape, ParallelConfig, RankPlacement  # noqa: E402

REF = C.CDLL(str(ROOT / "oracle" / "_ref" / "libcurator_ref.so"))
REF.ref_last_error.restype = C.c_char_p
_D, _PD = C.c_double, C.POINTER(C.c_double)
REF.ref_lr_at.argtypes = [_D, _PD]
REF.ref_batch_size_at.argtypes = [_D, C.POINTER(C.c_int32)]
REF.ref_weight_init_std.argtypes = [_D, _PD]
REF.ref_activation_bytes.argtypes = [_D, _D, _D, _D, _PD]
REF.ref_model_state_bytes.argtypes = [_D, _PD]
REF.ref_pipeline_efficiency.argtypes = [C.c_int32, C.c_int32, _PD]
REF.ref_estimated_tflops_per_gpu.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, _D, _PD]
REF.ref_plan_report.argtypes = [C.c_char_p, C.c_int32, C.c_char_p, C.c_int64, C.POINTER(C.c_int64)]
REF.ref_map_topology.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(C.c_int64)]


def topo(nodes, gpn, peak=312e12):
    return ClusterTopology(nodes, gpn, 600e9, 25e9, peak)


def ref_map(nodes, gpn, tp, pp, dp):
    n = C.c_int64()
    out = (RankPlacement * max(1, nodes * gpn))()
    t, p = topo(nodes, gpn), ParallelConfig(tp, pp, dp, 1, 1)
    rc = REF.ref_map_topology(C.byref(t), C.byref(p), out, len(out), C.byref(n))
    if rc:
        return {"error": rc, "message": REF.ref_last_error().decode()}
    return {"ranks": [[o.data, o.pipeline, o.tensor, o.node, o.gpu] for o in out[: n.value]]}


def f64(fn, *args):
    out = C.c_double()
    rc = fn(*args, C.byref(out))
    return {"error": rc, "message": REF.ref_last_error().decode()} if rc else out.value.hex()


def main():
    g = {"map_topology": [], "pipeline_efficiency": [], "lr_at": [], "batch_size_at": [], "weight_init_std": [],
         "activation_bytes": [], "model_state_bytes": [], "estimated_tflops_per_gpu": [], "plan_report": []}
    layouts = set()
    for gpus in (1, 2, 4, 8, 16):
        for tp in (1, 2, 4, 8, 16):
            for pp in (1, 2, 4, 8, 16):
                for dp in (1, 2, 4, 8, 16):
                    if tp * pp * dp == gpus:
                        layouts.add((1, gpus, tp, pp, dp))
    layouts |= {(280, 8, 8, 35, 8), (8, 8, 8, 2, 4), (1, 4, 2, 1, 2), (2, 8, 4, 2, 2),
                (1, 8, 16, 1, 1), (1, 8, 4, 1, 3), (1, 8, 3, 1, 1), (1, 8, 0, 1, 8), (2, 6, 4, 3, 1)}
    for L in sorted(layouts):
        g["map_topology"].append({"args": list(L), "out": ref_map(*L)})
    for mb in (1, 2, 4, 8, 16, 140, 280):
        for pp in (0, 1, 2, 4, 35):
            g["pipeline_efficiency"].append({"args": [mb, pp], "out": f64(REF.ref_pipeline_efficiency, mb, pp)})
    for t in (0.0, 5e8, 1e9 - 1, 1e9, 1e9 + 1, 1.71e11, 3.41e11, 1e12, -1.0):
        g["lr_at"].append({"args": [t.hex()], "out": f64(REF.ref_lr_at, t)})
    for t in (0.0, 2e8, 6e9, 1.2e10 - 1, 1.2e10, 5e11, -1.0):
        out = C.c_int32()
        rc = REF.ref_batch_size_at(t, C.byref(out))
        g["batch_size_at"].append({"args": [t.hex()], "out": out.value if rc == 0 else {"error": rc}})
    for h in (256.0, 1024.0, 8192.0, 12288.0, 20480.0, 1.0 / 3.0, 0.0):
        g["weight_init_std"].append({"args": [h.hex()], "out": f64(REF.ref_weight_init_std, h)})
    for a in ((4, 2, 128, 256), (1, 1, 2048, 20480), (1, 1, 2048, 12288), (1920, 105, 2048, 20480), (-1, 1, 1, 1)):
        g["activation_bytes"].append({"args": list(a), "out": f64(REF.ref_activation_bytes, *map(float, a))})
    for p in (0.0, 1.0, 175e9, 530e9, -1.0):
        g["model_state_bytes"].append({"args": [p.hex()], "out": f64(REF.ref_model_state_bytes, p)})
    shapes = [(530e9, 105, 20480, 128, 2048), (175e9, 96, 12288, 96, 2048), (0, 1, 12288, 96, 2048),
              (0, 1, 20480, 128, 2048), (0, 8, 8192, 64, 2048), (0, 2, 256, 4, 128)]
    for (P, L, h, H, s) in shapes:
        for (nodes, gpn, B, secs) in ((280, 8, 1920, 60.1), (350, 8, 1920, 50.2), (420, 8, 1920, 44.4),
                                      (1, 1, 1, 0.0265), (1, 8, 16, 0.2), (0, 8, 1, 1.0), (1, 8, 1, 0.0)):
            sh = ModelShape(P, L, h, H, s, 50257)
            t, par = topo(nodes, gpn), ParallelConfig(1, 1, 1, B, 1)
            g["estimated_tflops_per_gpu"].append({"args": [P, L, h, H, s, nodes, gpn, B, secs.hex()],
                                                  "out": f64(REF.ref_estimated_tflops_per_gpu, C.byref(sh),
                                                             C.byref(par), C.byref(t), secs)})
    configs = {
        "paper": "# paper-scale run\nparameters = 530e9\nlayers = 105\nhidden = 20480\nheads = 128\nsequence = 2048\n"
                 "vocab = 50257\ntensor_parallel = 8\npipeline_parallel = 35\ndata_parallel = 8\nbatch = 1920\n"
                 "micro_batches = 140\nnodes = 280\ngpus_per_node = 8\niteration_seconds = 60.1\n",
        "config5_3d": "layers = 4\nhidden = 12288\nheads = 96\nsequence = 2048\ntensor_parallel = 2\n"
                      "pipeline_parallel = 2\ndata_parallel = 2\nbatch = 16\nmicro_batches = 8\nnodes = 1\n"
                      "gpus_per_node = 8\npeak_tflops_per_gpu = 1704.1\n",
        "config4_pp": "layers = 8\nhidden = 8192\nheads = 64\nsequence = 2048\ntensor_parallel = 2\n"
                      "pipeline_parallel = 4\nbatch = 16\nmicro_batches = 16\nnodes = 1\ngpus_per_node = 8\n"
                      "peak_tflops_per_gpu = 1704.1\niteration_seconds = 0.25\nintra_node_bw = 900e9\n",
        "bad_syntax": "layers: 105\n",
        "bad_key": "warp_drive = 9\n",
        "bad_number": "layers = twelve\n",
        "bad_layout": "tensor_parallel = 16\nnodes = 1\ngpus_per_node = 8\n",
    }
    with tempfile.TemporaryDirectory() as d:
        for name, text in configs.items():
            path = os.path.join(d, "plan.txt")
            Path(path).write_text(text)
            entry = {"name": name, "config": text}
            for as_json in (0, 1):
                n = C.c_int64()
                buf = C.create_string_buffer(1 << 16)
                rc = REF.ref_plan_report(path.encode(), as_json, buf, len(buf), C.byref(n))
                key = "json" if as_json else "text"
                entry[key] = buf.value.decode() if rc == 0 else {"error": rc,
                                                                 "message": REF.ref_last_error().decode().replace(d, "<dir>")}
            g["plan_report"].append(entry)
    out = Path(__file__).with_name("planner_golden.json")
    out.write_text(json.dumps(g, indent=1) + "\n")
    print(f"wrote {out} ({sum(len(v) for v in g.values())} cases)")


if __name__ == "__main__":
    main()
