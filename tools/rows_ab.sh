# A/B: row kernels with one vs two resident CTAs per SM (MT_ROWS_MINB), launch lists of one bench step
# (GPT-3 h=12288 TP=1, and the MT-NLG TP=8 shard: h=20480 rows), plus the plain-copy ceiling.
python tools/copy_ceiling.py
python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
for m in 1 2; do
  MT_ROWS_MINB=$m ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 40 --csv --log-file gpurun_out/rows_minb$m.csv python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
  MT_ROWS_MINB=$m ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 40 --csv --log-file gpurun_out/rows_mt8_minb$m.csv python bench.py --config mtnlg --shard-of 8 --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
done
python - <<'PY'
import csv
for tag in ("", "mt8_"):
    for m in (1, 2):
        rows = list(csv.DictReader(l for l in open(f"gpurun_out/rows_{tag}minb{m}.csv") if l.startswith('"')))
        tot = 0
        for r in rows:
            name = r["Kernel Name"]
            t = float(r["Metric Value"].replace(",", ""))
            tot += t
            if any(k in name for k in ("ln_fwd_rows", "bdr_ln_rows", "ln_bwd_rows", "colsum")):
                print(tag or "gpt3_", "minb", m, name.split("(")[0][-60:], r["Metric Value"], r.get("Metric Unit"))
        print(tag or "gpt3_", "minb", m, "sum of launches", round(tot), flush=True)
PY
