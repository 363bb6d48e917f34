#!/bin/bash
# Fused (flash) vs unfused attention at the benchmarked shapes, alternating on one box, op timing on.
# Attention ops summed from the per-op breakdown.
set -u
for cfg in "" "--config mtnlg --shard-of 8" "--config gpt3 --shard-of 8"; do
for r in 1 2; do
for v in 0 1; do
  MT_ATTN_FUSED=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --op-timing $cfg 2>/dev/null | grep "^{" | \
  V=$v CFG="$cfg" python -c "
import json,sys,os
d=json.loads(sys.stdin.read()); b=d.get('op_breakdown_ms',{})
att=sum(v for k,v in b.items() if any(t in k for t in ('attn','softmax','flash')))
print(os.environ['CFG'] or 'default', 'fused=%s'%os.environ['V'], 'ms', round(d['ms_per_step'],3), 'attn_ops_ms', round(att,3), 'sm', d['clocks'].get('sm_mhz'), 'loss', d.get('loss'))"
done; done; done
