# Hidden-dropout keep bytes written by the forward bias-dropout-residual kernels and read by the
# backward's dropout' + bias-grad kernel, vs re-hashing: ncu durations of those kernels (MT-NLG TP=8
# shard and GPT-3 layer shapes) and the op-timing breakdown, alternating.
for r in 1 2; do
for v in 0 1; do
for cfg in "--config mtnlg --shard-of 8" "--config gpt3"; do
  MT_HIDDEN_KEEP=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --op-timing $cfg 2>/dev/null | grep "^{" | \
  V=$v C="$cfg" python -c "
import json,sys,os
d=json.loads(sys.stdin.read()); b=d.get('op_breakdown_ms',{})
print(os.environ['C'], 'keep=%s'%os.environ['V'], 'ms', round(d['ms_per_step'],3), {k: b.get(k) for k in ('fwd.bias_dropout_residual_ln','bwd.dropout_bias_grad')}, 'sm', d['clocks'].get('sm_mhz'))"
done; done; done
for v in 0 1; do
  MT_HIDDEN_KEEP=$v ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"bdr_|colsum_stage1|bias_dropout" -c 12 --csv \
    python bench.py --steps 1 --warmup 1 --no-cpu --config mtnlg --shard-of 8 2>/dev/null | grep gpu__time | awk -F'","' -v c="keep=$v" '{print c, substr($5,1,50), $NF}' | tail -6
done
