# plain bench (no per-op marks), unfused vs fused attention, alternating, 3 rounds
for r in 1 2 3; do
for v in "MT_ATTN_FUSED=0" "MT_ATTN_FUSED=1"; do
  env $v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/ab.json 2>&1
  python -c "
import json
d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
print('$v', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],3), 'sm', d['clocks']['sm_mhz'], 'loss', round(d['loss'],5))"
done; done
