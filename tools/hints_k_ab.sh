# A/B: L2 eviction hints on the short-K (<= 16384) m-fastest GEMMs (default) vs plain loads for every
# m-fastest GEMM (MT_GEMM_SHORTK_HINTS=0): launch lists of one GPT-3 bench step and bench steps.
python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
for v in 0 1; do
  MT_GEMM_SHORTK_HINTS=$v ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 40 --csv --log-file gpurun_out/hk_$v.csv python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
done
python - <<'PY'
import csv
a = [r for r in csv.DictReader(l for l in open("gpurun_out/hk_0.csv") if l.startswith('"'))]
b = [r for r in csv.DictReader(l for l in open("gpurun_out/hk_1.csv") if l.startswith('"'))]
ta = tb = 0
for x, y in zip(a, b):
    va, vb = float(x["Metric Value"].replace(",", "")), float(y["Metric Value"].replace(",", ""))
    ta += va; tb += vb
    if "gemm" in x["Kernel Name"]:
        print(f'{x["Kernel Name"].split("(")[0][-40:]:40s} {va/1e3:9.1f} {vb/1e3:9.1f}')
print("sum of launches plain / short-K hints", round(ta / 1e3), round(tb / 1e3))
PY
for r in 1 2; do
  for v in 0 1; do
    MT_GEMM_SHORTK_HINTS=$v python bench.py --steps 20 --warmup 5 --no-cpu | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench shortk_hints=$v', round(d['ms_per_step'],3), d['clocks']['sm_mhz'], d['clocks'].get('power_w_max'))"
  done
done
for cfg in "--config gpt3 --shard-of 4" "--config mtnlg --shard-of 8"; do
  for v in 0 1; do
    MT_GEMM_SHORTK_HINTS=$v python bench.py --steps 20 --warmup 5 --no-cpu $cfg | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$cfg shortk_hints=$v', round(d['ms_per_step'],3), d['clocks']['sm_mhz'])"
  done
done
