# same-box A/B of the split-K threshold on whole-layer benches (old behaviour: MT_GEMM_SPLIT_MINK=1)
for rep in 1 2; do
for cfg in "--shard-of 8" "--shard-of 8 --config mtnlg" "--shard-of 4" "--shard-of 4 --config mtnlg" ""; do
  for mink in 1 256; do
    MT_GEMM_SPLIT_MINK=$mink python bench.py $cfg --steps 10 --warmup 3 --no-cpu 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg'.ljust(28), 'mink=$mink', round(d['ms_per_step'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done
done
