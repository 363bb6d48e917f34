# Fused vs unfused attention at the MT-NLG TP=8 shard shape (hd 160), alternating, op timing on.
for r in 1 2 3; do
for v in 0 1; do
  MT_ATTN_FUSED=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --op-timing --config mtnlg --shard-of 8 2>/dev/null | grep "^{" | \
  V=$v python -c "
import json,sys,os
d=json.loads(sys.stdin.read()); b=d.get('op_breakdown_ms',{})
att=sum(v for k,v in b.items() if any(t in k for t in ('attn','softmax','flash')))
print('mtnlg shard-of-8 fused=%s'%os.environ['V'], 'ms', round(d['ms_per_step'],3), 'attn_ops_ms', round(att,3), 'sm', d['clocks'].get('sm_mhz'))"
done; done
