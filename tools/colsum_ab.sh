# column-reduction kernels: op timing at the TP=8 / TP=4 shard shapes for rows-per-split choices
for per in 64 86 128; do
  for cfg in "--shard-of 8" "--shard-of 4"; do
    MT_COL_ROWS_PER_SPLIT=$per python bench.py $cfg --steps 10 --warmup 3 --no-cpu --op-timing 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); o=d['op_breakdown_ms']; print('per=$per', '$cfg'.ljust(14), round(d['ms_per_step'],3), 'drop_bias', o['bwd.dropout_bias_grad'], 'bias', o['bwd.bias_grad'], 'lnb', o['bwd.ln_bwd'])"
  done
done
