# Ring depth of the TMA-fed row kernels (MT_ROW_STAGES): ncu durations at the GPT-3 (h 12288, whole
# rows) and MT-NLG TP=8 shard (h 20480, rows split over a 2-CTA cluster) shapes.
for cfg in "--config gpt3" "--config mtnlg --shard-of 8"; do
for st in 3 4 5 6; do
  MT_ROW_STAGES=$st ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"_rows_kernel" -c 6 --csv \
    python bench.py --steps 1 --warmup 1 --no-cpu $cfg 2>/dev/null | grep gpu__time | \
    awk -F'","' -v c="$cfg stages=$st" '{print c, substr($5,1,45), $NF}'
done; done
