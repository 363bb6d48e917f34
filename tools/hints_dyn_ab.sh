# A/B with the dynamic tile scheduler: L2 eviction hints on the m-fastest GEMMs (MT_GEMM_HINTS unset =
# none for them; 1 = A evict_last + B evict_first; 2 = A evict_last only). Standalone rates, DRAM bytes,
# launch lists of one GPT-3 bench step, bench steps.
run_h() { local h=$1; shift; if [ -z "$h" ]; then env -u MT_GEMM_HINTS "$@"; else MT_GEMM_HINTS=$h "$@"; fi; }
for g in fc1_fwd fc1_dgrad fc2_fwd qkv_fwd; do
  for h in "" 1 2; do echo "hints=${h:-default} $(run_h "$h" python tools/gemm_one.py $g 8 | tail -1)"; done
done
for g in fc1_fwd fc1_dgrad fc2_fwd; do
  for h in "" 1 2; do
    run_h "$h" ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none \
      -k regex:gemm_sm100 -s 2 -c 1 --csv python tools/gemm_one.py $g 3 2>/dev/null | grep 'dram__\|gpu__time' | \
      awk -F'","' -v g=$g -v h=${h:-default} '{print "ncu", g, "hints=" h, $(NF-2), $NF}'
  done
done
python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
for h in "" 1; do
  run_h "$h" ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 40 --csv --log-file gpurun_out/hdyn_${h:-d}.csv python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
done
python - <<'PY'
import csv
for f in ("d", "1"):
    rows = [r for r in csv.DictReader(l for l in open(f"gpurun_out/hdyn_{f}.csv") if l.startswith('"'))]
    print("hints", f, "sum of launches", round(sum(float(r["Metric Value"].replace(",", "")) for r in rows) / 1e3))
PY
for r in 1 2; do
  for h in "" 1; do
    run_h "$h" python bench.py --steps 20 --warmup 5 --no-cpu | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench hints=${h:-default}', round(d['ms_per_step'],3), d['clocks']['sm_mhz'], d['clocks'].get('power_w_max'))"
  done
done
