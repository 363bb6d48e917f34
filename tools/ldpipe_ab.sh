# A/B: software-pipelined accumulator reads in the GEMM epilogue vs one load-wait-process per piece
# (MT_GEMM_NO_LDPIPE=1, compile-time): launch lists of one GPT-3 bench step each.
python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 40 --csv --log-file gpurun_out/ab_ldpipe.csv python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
MT_NVCC_DEFINES="-DMT_GEMM_NO_LDPIPE=1" python -m paper_2201_11990_b200.build > /dev/null
ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 40 --csv --log-file gpurun_out/ab_noldpipe.csv python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
python -m paper_2201_11990_b200.build > /dev/null
python - <<'PY'
import csv
a = [r for r in csv.DictReader(l for l in open("gpurun_out/ab_noldpipe.csv") if l.startswith('"'))]
b = [r for r in csv.DictReader(l for l in open("gpurun_out/ab_ldpipe.csv") if l.startswith('"'))]
ta = tb = 0
for x, y in zip(a, b):
    va, vb = float(x["Metric Value"].replace(",", "")), float(y["Metric Value"].replace(",", ""))
    ta += va; tb += vb
    print(f'{x["Kernel Name"].split("(")[0][-55:]:55s} {va/1e3:9.1f} {vb/1e3:9.1f}')
print("sum", round(ta / 1e3), round(tb / 1e3))
PY
