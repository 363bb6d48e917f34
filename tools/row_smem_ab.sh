# Row-kernel ring budget (MT_ROW_SMEM_KB): 200 KB (2 stages of dy/x/resid rows at h = 12288 in the
# LayerNorm backward) vs 224 KB (3 stages): ncu durations at the GPT-3 and MT-NLG TP=8 shard shapes.
for r in 1 2; do
for kb in 200 224; do
for cfg in "--config gpt3" "--config mtnlg --shard-of 8"; do
  MT_ROW_SMEM_KB=$kb ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"_rows_kernel" -c 6 --csv \
    python bench.py --steps 1 --warmup 1 --no-cpu $cfg 2>/dev/null | grep gpu__time | \
    awk -F'","' -v c="$cfg kb=$kb" '{print c, substr($5,1,45), $NF}'
done; done; done
