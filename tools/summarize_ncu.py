"""Summarise ncu outputs in gpurun_out/ into profiles/<round>_*.md (+ profiles/gemm_traffic.json).

    python tools/summarize_ncu.py r01
"""
import collections
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "gpurun_out"
PROF = ROOT / "profiles"
PROF.mkdir(exist_ok=True)
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]


def raw(rep):
    r = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True)
    rows = list(csv.reader(io.StringIO(r.stdout)))
    if len(rows) < 3:
        return []
    hdr, units = rows[0], rows[1]
    out = []
    for row in rows[2:]:
        d = {}
        for key, label in METRICS:
            if key in hdr:
                i = hdr.index(key)
                d[label] = f"{row[i]} {units[i]}".strip()
                d[key] = (row[i], units[i])
        d["kernel"] = row[hdr.index("Kernel Name")][:100]
        out.append(d)
    return out


def to_bytes(v):
    val, unit = v
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return float(val.replace(",", "")) * mult


lines = [f"# {tag}: ncu summaries (B200, `--clock-control none`)\n"]
# 1. launch list
lc = OUT / "launches.csv"
if lc.exists():
    rows = [r for r in csv.reader(open(lc)) if r]
    hdr = next(r for r in rows if r[0] == "ID")
    data = [dict(zip(hdr, r)) for r in rows if len(r) == len(hdr) and r[0] != "ID"]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        if d["Metric Name"] == "gpu__time_duration.sum":
            k = d["Kernel Name"].split("(")[0][:80]
            agg[k][0] += 1
            agg[k][1] += float(d["Metric Value"])
    tot = sum(v[1] for v in agg.values())
    lines.append("## Launch list of `python bench.py --steps 2 --warmup 3 --no-cpu` (gpu__time_duration.sum)\n")
    lines.append("Cold-cache, serialised replay: compare shares, not absolutes. Includes warmup, init and e2e steps.\n")
    lines.append("| share | launches | avg us | kernel |\n|---:|---:|---:|---|")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| {100 * v[1] / tot:.1f}% | {v[0]} | {v[1] / v[0] / 1e3:.1f} | `{k}` |")
    lines.append("")
traffic = {}
for rep in sorted(OUT.glob("prof_gemm_*.ncu-rep")) + sorted(OUT.glob("prof_hbm.ncu-rep")):
    res = raw(rep)
    if not res:
        continue
    lines.append(f"## `{rep.name}` (--set full)\n")
    lines.append("| kernel | " + " | ".join(l for _, l in METRICS) + " |")
    lines.append("|---|" + "---|" * len(METRICS))
    for d in res:
        lines.append(f"| `{d['kernel'][:60]}` | " + " | ".join(d.get(l, "") for _, l in METRICS) + " |")
        if "gemm" in rep.name and "dram__bytes_read.sum" in d:
            traffic[rep.stem] = to_bytes(d["dram__bytes_read.sum"]) + to_bytes(d["dram__bytes_write.sum"])
    lines.append("")
(PROF / f"{tag}_ncu_summary.md").write_text("\n".join(lines) + "\n")
if traffic:
    (PROF / "gemm_traffic.json").write_text(json.dumps({
        "source": f"profiles/{tag}_ncu_summary.md (ncu --set full, one launch each)",
        "dram_bytes_per_launch": traffic.get("prof_gemm_fc1_fwd"),
        "per_gemm": traffic}, indent=1) + "\n")
print((PROF / f"{tag}_ncu_summary.md").read_text()[:3000])
