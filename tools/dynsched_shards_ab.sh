# A/B of the dynamic tile scheduler at the TP-shard shapes: single-GPU shard benches (compute only)
# and the shard GEMMs standalone, static (MT_GEMM_DYNAMIC=0) vs dynamic, alternating.
for r in 1 2; do
  for cfg in "--config gpt3 --shard-of 4" "--config gpt3 --shard-of 8" "--config mtnlg --shard-of 8" "--config mtnlg --shard-of 4"; do
    for d in 0 1; do
      MT_GEMM_DYNAMIC=$d python bench.py --steps 20 --warmup 5 --no-cpu $cfg | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$cfg dyn=$d', round(d['ms_per_step'],3), round(d['roofline']['achieved']), d['clocks']['sm_mhz'], d['clocks'].get('power_w_max'))"
    done
  done
done
for g in g4_proj_fwd g8_proj_fwd g8_fc2_fwd fc2_fwd_g4 qkv_dgrad_g4 g8_qkv_dgrad fc1_wgrad_g8 mt_fc1_fwd mt_fc2_fwd mt_proj_fwd mt_fc1_wgrad; do
  for d in 0 1; do echo "dyn=$d $(MT_GEMM_DYNAMIC=$d python tools/gemm_one.py $g 8 | tail -1)"; done
done
