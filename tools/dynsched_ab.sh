# A/B: dynamic tile scheduler (default) vs static round-robin (MT_GEMM_DYNAMIC=0): standalone GEMM
# rates, DRAM bytes per launch (ncu), launch lists of one GPT-3 bench step, and bench steps.
for g in fc1_fwd fc1_dgrad fc2_fwd qkv_fwd fc1_wgrad; do
  for d in 0 1; do echo "dyn=$d $(MT_GEMM_DYNAMIC=$d python tools/gemm_one.py $g 8 | tail -1)"; done
done
for g in fc1_fwd fc1_dgrad fc1_wgrad; do
  for d in 0 1; do
    MT_GEMM_DYNAMIC=$d ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -k regex:gemm_sm100 -s 2 -c 1 --csv python tools/gemm_one.py $g 3 2>/dev/null | grep '"gemm_sm100\|dram__\|gpu__time' | \
      awk -F'","' -v g=$g -v d=$d '{print "ncu", g, "dyn=" d, $(NF-2), $NF}'
  done
done
python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
for d in 0 1; do
  MT_GEMM_DYNAMIC=$d ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 40 --csv --log-file gpurun_out/dyn_$d.csv python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
done
python - <<'PY'
import csv
a = [r for r in csv.DictReader(l for l in open("gpurun_out/dyn_0.csv") if l.startswith('"'))]
b = [r for r in csv.DictReader(l for l in open("gpurun_out/dyn_1.csv") if l.startswith('"'))]
ta = tb = 0
for x, y in zip(a, b):
    va, vb = float(x["Metric Value"].replace(",", "")), float(y["Metric Value"].replace(",", ""))
    ta += va; tb += vb
    if "gemm" in x["Kernel Name"]:
        print(f'{x["Kernel Name"].split("(")[0][-40:]:40s} {va/1e3:9.1f} {vb/1e3:9.1f}')
print("sum of launches static / dynamic", round(ta / 1e3), round(tb / 1e3))
PY
for r in 1 2; do
  for d in 0 1; do
    MT_GEMM_DYNAMIC=$d python bench.py --steps 20 --warmup 5 --no-cpu | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench dyn=$d', round(d['ms_per_step'],3), d['clocks']['sm_mhz'], d['clocks'].get('power_w_max'))"
  done
done
