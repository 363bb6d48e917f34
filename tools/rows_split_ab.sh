# A/B: row kernels with whole rows per CTA (MT_ROWS_SPLIT=1) vs rows split over a 2-CTA cluster
# (default for h >= 8192): launch lists of one bench step, GPT-3 h=12288 TP=1 and the MT-NLG TP=8 shard.
python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
for m in 1 auto; do
  MT_ROWS_SPLIT=$m ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 40 --csv --log-file gpurun_out/rsplit_gpt3_$m.csv python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
  MT_ROWS_SPLIT=$m ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 40 --csv --log-file gpurun_out/rsplit_mt8_$m.csv python bench.py --config mtnlg --shard-of 8 --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
done
python - <<'PY'
import csv
for tag in ("gpt3", "mt8"):
    for m in ("1", "auto"):
        rows = list(csv.DictReader(l for l in open(f"gpurun_out/rsplit_{tag}_{m}.csv") if l.startswith('"')))
        tot = 0
        for r in rows:
            name = r["Kernel Name"]
            t = float(r["Metric Value"].replace(",", ""))
            tot += t
            if any(k in name for k in ("ln_fwd_rows", "bdr_ln_rows", "ln_bwd_rows", "colsum")):
                print(tag, "split", m, name.split("(")[0][-50:], r["Metric Value"], flush=True)
        print(tag, "split", m, "sum of launches", round(tot), flush=True)
PY
