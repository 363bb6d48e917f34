#!/usr/bin/env python
"""Benchmark of the MT-NLG tensor-sliced training step on B200 (driver contract: one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config gpt3|mtnlg|pp|3d|tiny] [--impl ours|reference]

N > 1 is launched by the driver through torch.distributed.run (one rank per GPU; RANK/LOCAL_RANK/
WORLD_SIZE/MASTER_* from the env). A step is one training iteration of the configured layout through
the runtime's public API (mt_stage_train_step*): zero grads, 1F1B over the microbatches (layer
forward + backward on the sm_100a kernels, TP all-reduces, PP send/recv), synthetic MSE loss, DP
gradient all-reduce.

Default config (BASELINE.json configs[1]): one GPT-3-175B-shape layer (h=12288, 96 heads, s=2048,
b=1) with TP = N. value = whole-job tokens/s (b*s*MB*DP / step time, max over ranks, device
resident inputs); e2e = the same through host (pinned) input/target buffers with the H2D copies
and the loss D2H inside the timed region. Algorithmic FLOPs per GPU = 72*b*s*h^2*(1+s/(6h)) *
layers_per_stage * MB / TP (the reference cost model proj/src/planner.cpp:52-54 with V=0, no
recompute).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "TFLOP/s/GPU & tokens/s, tensor-sliced layer fwd+bwd, 1/2/4/8 B200"
SEED = 20260808


def layout_for(config: str, n: int) -> dict:
    """Model shape + (TP, PP, DP) for `config` on n GPUs (per-GPU shapes kept when n < 8)."""
    if config == "gpt3":
        return dict(hidden=12288, heads=96, seq=2048, b=1, layers=1, mb=1, tp=n, pp=1, dp=1,
                    model="GPT-3-175B-shape layer", note=f"TP={n}")
    if config == "mtnlg":
        return dict(hidden=20480, heads=128, seq=2048, b=1, layers=1, mb=1, tp=n, pp=1, dp=1,
                    model="MT-NLG-530B-shape layer", note=f"TP={n}")
    if config == "dp":  # h=8192 2-layer slice replicated over DP = n, 4 microbatches per replica
        return dict(hidden=8192, heads=64, seq=2048, b=1, layers=2, mb=4, tp=1, pp=1, dp=n,
                    model="h=8192 2-layer slice, data parallel", note=f"DP={n} (MB=4)")
    if config == "tiny":
        return dict(hidden=256, heads=4, seq=128, b=4, layers=2, mb=1, tp=n, pp=1, dp=1,
                    model="tiny GPT (2 layers, h=256)", note=f"TP={n}")
    if config == "pp":  # 8-layer h=8192 slice, PP=4 x TP=2, 16 microbatches (2 layers per stage kept)
        tp = 2 if n >= 2 else 1
        pp = max(1, n // tp)
        return dict(hidden=8192, heads=64, seq=2048, b=1, layers=2 * pp, mb=16, tp=tp, pp=pp, dp=1,
                    model="h=8192 slice, 1F1B", note=f"PP={pp} x TP={tp} ({2 * pp} layers)")
    if config == "3d":  # 4-layer h=12288 slice, DP=2 x PP=2 x TP=2, 8 microbatches
        tp = 2 if n >= 2 else 1
        pp = 2 if n >= 4 else 1
        dp = max(1, n // (tp * pp))
        return dict(hidden=12288, heads=96, seq=2048, b=1, layers=2 * pp, mb=8, tp=tp, pp=pp, dp=dp,
                    model="h=12288 slice, 3D", note=f"DP={dp} x PP={pp} x TP={tp} ({2 * pp} layers)")
    raise SystemExit(f"unknown config {config}")


def algorithmic_flops_per_gpu(L: dict) -> float:
    h, s = L["hidden"], L["seq"]
    per_layer = 72.0 * L["b"] * s * h * h * (1.0 + s / (6.0 * h))
    return per_layer * (L["layers"] // L["pp"]) * L["mb"] / L["tp"]


def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"bf16": d["bf16_tflops"], "bf16_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]),
                "hbm": d["hbm_gbs"], "source": "measured"}
    return {"bf16": 1590.0, "bf16_sustained": 1400.0, "hbm": 6650.0, "source": "fallback"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons, sampled every 50 ms from before the warm-up steps to after the
    timed region; summary() reports the samples that fall inside the timed window (mark_start/mark_end),
    widened to the last 2 s before its end when the window is too short for 3 samples (the warm-up steps
    run the same workload)."""
    FIELDS = ["timestamp", "clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.t0 = self.t1 = None
        self.out = ""

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={','.join(self.FIELDS)}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        time.sleep(0.2)
        return self

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()

    def stop(self):
        if self.proc:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    @staticmethod
    def _ts(text: str):
        from datetime import datetime
        try:
            return datetime.strptime(text.strip(), "%Y/%m/%d %H:%M:%S.%f").timestamp()
        except ValueError:
            return None

    def summary(self) -> dict:
        rows = []
        for line in (self.out or "").splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == len(self.FIELDS):
                rows.append((self._ts(parts[0]), parts[1:]))
        window = "timed region"
        sel = [r for t, r in rows if t is not None and self.t0 and self.t1 and self.t0 - 0.05 <= t <= self.t1 + 0.05]
        if len(sel) < 3 and self.t1:
            sel = [r for t, r in rows if t is not None and self.t1 - 2.0 <= t <= self.t1 + 0.05]
            window = "last 2 s before the end of the timed region (warm-up + timed steps)"
        if not sel:
            sel, window = [r for _, r in rows], "whole run"
        if not sel:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in sel if r[0].replace(".", "").isdigit()]
        loaded = [v for v in sm if v > 500] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in sel for i in range(4) if r[3 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": float(sel[0][1]) if sel[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(sel), "window": window,
                "power_w_max": max(float(r[2]) for r in sel if r[2].replace(".", "").isdigit())}


# ----------------------------------------------------------------------------------------------- CPU arm
def cpu_sample(L: dict, steps: int, warmup: int, threads_note: str = "") -> dict:
    """The CPU restatement (oracle/layer_oracle.cpp, OpenMP over all host cores) on a bounded sample
    of the same workload: one layer of the configured shape, fwd+bwd, on a short token sample."""
    import numpy as np
    from oracle import oracle as O
    h, H = L["hidden"], L["heads"]
    tokens = min(L["seq"], 128)
    rng = np.random.default_rng(0)
    std = 1.0 / np.sqrt(3.0 * h)
    base = rng.standard_normal(1 << 20, dtype=np.float32)  # values do not change the timing: tile one block
    params = []
    for i, (r, c) in enumerate(O.param_shapes(h)):
        a = np.resize(base, (r, c))
        a *= np.float32(std if i in O.WEIGHTS else 0.02)
        if i in O.GAMMAS:
            a += np.float32(1.0)
        params.append(a)
    ol = O.OracleLayer(h, H, tokens, 1, 1, dropout_hidden=0.1, dropout_attn=0.1, bf16_emulate=False,
                       params=params)
    x = rng.standard_normal((tokens, h), dtype=np.float32)
    g = rng.standard_normal((tokens, h), dtype=np.float32) * 1e-3
    times = []
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        ol.forward(x, i)
        ol.backward(g, i)
        if i >= warmup:
            times.append(time.perf_counter() - t0)
    t = statistics.median(times)
    return {"value": tokens / t, "unit": "tokens/s", "cores": O.num_threads(), "kind": "port",
            "sample": f"1 layer h={h} heads={H}, {tokens}-token sequence (of {L['seq']}), fwd+bwd fp32, "
                      f"median of {steps} after {warmup} warmup; oracle/layer_oracle.cpp (the reference has no "
                      f"layer implementation: SPEC.md:8)",
            "seconds_per_sample": t}


def run_reference(args, L: dict) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    # rank 0 alone runs the CPU reference: give it every host thread (torchrun exports OMP_NUM_THREADS=1;
    # the OpenMP runtime reads it when the oracle library loads, which happens below)
    os.environ["OMP_NUM_THREADS"] = str(os.cpu_count() or 1)
    steps = max(1, min(args.steps, 5))
    warmup = max(1, min(args.warmup, 2))
    cb = cpu_sample(L, steps, warmup)
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "tokens/s",
            "n_gpus": args.gpus, "steps": steps, "warmup": warmup, "ms_per_step": 1e3 * cb["seconds_per_sample"],
            "higher_is_better": True, "scaling": "strong" if L["dp"] == 1 else "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{L['model']} {L['note']} (CPU sample)", "hidden": L["hidden"],
                       "heads": L["heads"], "seq_len": L["seq"]},
            "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": cb["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------------------------- GPU arm
def run_ours(args, L: dict) -> None:
    import torch
    import torch.distributed as dist
    from paper_2201_11990_b200 import planner as PL
    from paper_2201_11990_b200._native import lib
    from paper_2201_11990_b200.runtime import Context, Stage

    lib()  # fail loudly if the native library is missing
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    shard_only = L.get("shard_only", False)
    if not shard_only and world != L["tp"] * L["pp"] * L["dp"]:
        raise SystemExit(f"layout {L['note']} needs {L['tp'] * L['pp'] * L['dp']} ranks, got {world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = Context(local)
    if world > 1:
        obj = [Context.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ctx.init_comm(obj[0], world, rank, L["tp"], L["pp"], L["dp"], L["b"] * L["mb"] * L["dp"], L["mb"])
    else:
        ctx.init_comm(bytes(128), 1, 0, 1, 1, 1, L["b"] * L["mb"], L["mb"])
    if shard_only:
        lib().mt_ctx_shard_only(ctx._h, 1)
    place = ctx.placement()
    first, last = place.pipeline == 0, place.pipeline == L["pp"] - 1
    desc = PL.layer_desc(L["hidden"], L["heads"], L["seq"], L["b"], dropout_hidden=args.dropout,
                         dropout_attn=args.dropout,
                         seed=SEED, tp_size=L["tp"] if shard_only else 1)
    stage = Stage(ctx, desc, L["layers"], L["mb"])
    if args.recompute:
        stage.set_recompute(True)
    stream = torch.cuda.current_stream()
    stage.init_params(L["layers"] // L["pp"], stream)
    M, h, MB = L["b"] * L["seq"], L["hidden"], L["mb"]
    gen = torch.Generator(device="cuda").manual_seed(SEED + place.data)
    x_dev = torch.randn(MB, M, h, device="cuda", generator=gen).bfloat16() if first else None
    t_dev = torch.randn(MB, M, h, device="cuda", generator=gen).bfloat16() if last else None
    loss_dev = torch.zeros(1, device="cuda")

    def step_dev():
        stage.train_step_dev(x_dev.data_ptr() if first else 0, t_dev.data_ptr() if last else 0,
                             loss_dev.data_ptr(), stream)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    clk = ClockSampler(local).start()  # sampling from before the warm-up (clocks settle under load)
    for _ in range(args.warmup):
        step_dev()
    torch.cuda.synchronize()
    launches_per_step = stage.launch_count()

    # ---- device-resident timed region (per-GEMM events on for the live roofline)
    lib().mt_ctx_gemm_timing(ctx._h, 1)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    clk.mark_start()
    ev0.record(stream)
    for _ in range(args.steps):
        step_dev()
    ev1.record(stream)
    torch.cuda.synchronize()
    clk.mark_end()
    barrier()
    clk.stop()
    import ctypes as C
    g_ms, g_fl, g_n = C.c_double(), C.c_double(), C.c_int64()
    lib().mt_ctx_gemm_timing_read(ctx._h, C.byref(g_ms), C.byref(g_fl), C.byref(g_n))
    lib().mt_ctx_gemm_timing(ctx._h, 0)
    ms = max_over_ranks(ev0.elapsed_time(ev1) / args.steps)
    loss_value = float(loss_dev.item())

    # ---- end-to-end through host buffers (pinned): H2D inputs/targets + loss D2H inside the region
    x_host = x_dev.cpu().pin_memory() if first else None
    t_host = t_dev.cpu().pin_memory() if last else None
    h2d = (x_host.numel() * 2 if first else 0) + (t_host.numel() * 2 if last else 0)
    d2h = 4 if last else 0
    stage.train_step(x_host.data_ptr() if first else None, t_host.data_ptr() if last else None, stream)
    torch.cuda.synchronize()
    barrier()
    t0 = time.perf_counter()
    ev0.record(stream)
    for _ in range(args.steps):
        stage.train_step(x_host.data_ptr() if first else None, t_host.data_ptr() if last else None, stream)
    ev1.record(stream)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / args.steps * 1e3
    e2e_ms = max_over_ranks(max(ev0.elapsed_time(ev1) / args.steps, wall))
    h2d, d2h = stage.host_traffic()  # bytes actually moved (TP ranks copy 1/TP slices each)
    tot = torch.tensor([h2d, d2h], device="cuda", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(tot)
    h2d_all, d2h_all = int(tot[0].item()), int(tot[1].item())

    # optimizer step, timed separately: the metric is the layer fwd+bwd
    from paper_2201_11990_b200.runtime import adam_defaults
    adam = adam_defaults(tokens_seen=1e10, step=1)
    stage.optimizer_step(adam, stream, want_norm=False)
    torch.cuda.synchronize()
    ev0.record(stream)
    for i in range(args.steps):
        adam.step = 2 + i
        stage.optimizer_step(adam, stream, want_norm=False)
    ev1.record(stream)
    torch.cuda.synchronize()
    opt_ms = max_over_ranks(ev0.elapsed_time(ev1) / args.steps)
    op_breakdown = None
    if args.op_timing:
        lib().mt_ctx_op_timing(ctx._h, 1)
        for _ in range(args.steps):
            step_dev()
        buf = C.create_string_buffer(1 << 16)
        n = C.c_int64()
        lib().mt_ctx_op_timing_read(ctx._h, buf, len(buf), C.byref(n))
        lib().mt_ctx_op_timing(ctx._h, 0)
        op_breakdown = {}
        for line in buf.value.decode().splitlines():
            name, tot, cnt = line.split()
            op_breakdown[name] = round(float(tot) / args.steps, 4)
        if world > 1:
            allb = [None] * world
            dist.all_gather_object(allb, op_breakdown)
            op_breakdown = {f"rank{r}": b for r, b in enumerate(allb)}
    clocks = clk.summary()
    pk = peaks()
    tokens = L["b"] * L["seq"] * MB * L["dp"]
    flops_gpu = algorithmic_flops_per_gpu(L)
    tflops_gpu = flops_gpu / (ms * 1e-3) / 1e12
    gemm_tflops = (g_fl.value / (g_ms.value * 1e-3) / 1e12) if g_ms.value > 0 else None
    traffic = None
    prof = ROOT / "profiles" / "gemm_traffic.json"
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    # the measured burst peak is the denominator for a timed region shorter than ~1 s (the sustained
    # figure is a seconds-long loop under the power cap)
    region_s = ms * args.steps * 1e-3
    peak_used = pk["bf16"] if region_s < 1.0 else pk["bf16_sustained"]
    peak_kind = (f"{pk['source']} burst bf16 (timed region {region_s:.2f} s < 1 s)" if region_s < 1.0 else
                 f"{pk['source']} sustained bf16 (timed region {region_s:.2f} s >= 1 s)")
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cpu = cpu_sample(L, 2, 1)
            cpu.pop("seconds_per_sample", None)
        except Exception as e:  # the CPU leg is a reported baseline; never fail the GPU bench on it
            cpu = {"value": None, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "port", "sample": f"failed: {e}"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": tokens / (ms * 1e-3), "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if L["dp"] == 1 else "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (seeded N(0,1) inputs/targets, seeded N(0, sqrt(1/3h)) weights)",
            "config": {"workload": f"{L['model']} fwd+bwd, {L['note']}", "hidden": L["hidden"], "heads": L["heads"],
                       "seq_len": L["seq"], "micro_batch": L["b"], "micro_batches": MB, "layers": L["layers"],
                       "global_batch": L["b"] * MB * L["dp"], "parallelism": f"tp{L['tp']}pp{L['pp']}dp{L['dp']}",
                       "dropout": args.dropout, "l2": "working set > L2 (weights alone exceed 126 MB); no flush"},
            "tflops_per_gpu": tflops_gpu,
            **({"recompute": True, "hardware_tflops_per_gpu": tflops_gpu * 96.0 / 72.0} if args.recompute else {}),
            "peak_fraction": tflops_gpu / pk["bf16"],
            "peak_fraction_sustained": tflops_gpu / pk["bf16_sustained"],
            "peak_fraction_datasheet": tflops_gpu / 2250.0,
            "tokens_per_s_per_gpu": tokens / (ms * 1e-3) / world,
            "loss": loss_value,
            "optimizer_ms_per_step": opt_ms,
            "roofline": {"bound": "tensor", "kernel": "gemm_sm100_kernel (tcgen05, all GEMM launches of the step)",
                         "achieved": gemm_tflops, "peak": peak_used, "unit": "TFLOP/s",
                         "frac": (gemm_tflops / peak_used) if gemm_tflops else None,
                         "frac_vs_burst": (gemm_tflops / pk["bf16"]) if gemm_tflops else None,
                         "frac_vs_sustained": (gemm_tflops / pk["bf16_sustained"]) if gemm_tflops else None,
                         "peak_kind": peak_kind,
                         "gemm_share_of_step": (g_ms.value / args.steps) / ms if ms else None,
                         "gemm_launches_per_step": g_n.value // max(args.steps, 1),
                         "traffic": traffic},
            "e2e": {"value": tokens / (e2e_ms * 1e-3), "unit": "tokens/s", "h2d_bytes_per_step": h2d_all,
                    "d2h_bytes_per_step": d2h_all, "ms_per_step": e2e_ms},
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks,
            "cpu_baseline": cpu,
            **({"shard_only": True} if shard_only else {}),
            **({"op_breakdown_ms": op_breakdown} if op_breakdown is not None else {}),
        }
        print(json.dumps(line), flush=True)
    stage.close()
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="gpt3", choices=["gpt3", "mtnlg", "pp", "3d", "dp", "tiny"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU-baseline leg")
    ap.add_argument("--dropout", type=float, default=0.1, help="hidden and attention dropout (Megatron default 0.1)")
    ap.add_argument("--shard-of", type=int, default=0,
                    help="single GPU: run ONE rank's tensor-parallel shard of the config at TP=SHARD_OF with the "
                         "TP all-reduces skipped (compute-only per-GPU measurement, flagged in the JSON)")
    ap.add_argument("--recompute", action="store_true",
                    help="activation recompute (SURVEY.md §8f N2): the backward re-runs each layer's forward; "
                         "tflops_per_gpu stays model FLOPs (72 coeff.), hardware_tflops_per_gpu counts the re-run (96)")
    ap.add_argument("--op-timing", action="store_true",
                    help="after the timed region, run the steps again with per-op event marks and report the "
                         "per-op breakdown (ms per step) in the JSON line as op_breakdown_ms")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    L = layout_for(args.config, args.gpus)
    if args.shard_of > 1:
        if args.gpus != 1 or int(os.environ.get("WORLD_SIZE", "1")) != 1:
            raise SystemExit("--shard-of is a single-GPU measurement")
        L = dict(L, tp=args.shard_of, shard_only=True,
                 note=f"ONE TP={args.shard_of} shard on 1 GPU, compute only (TP all-reduces excluded)")
    if args.impl == "reference":
        run_reference(args, L)
    else:
        run_ours(args, L)


if __name__ == "__main__":
    main()
