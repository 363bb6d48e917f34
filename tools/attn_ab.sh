timeout 300 python -m pytest tests/test_layer_gpu.py -q -x -p no:cacheprovider -k "flash or recompute" 2>&1 | tail -3
for v in "MT_ATTN_FUSED=0" "MT_ATTN_FUSED=1" "MT_ATTN_FUSED=1 MT_ATTN_FWD2=0"; do
  env $v timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --op-timing > gpurun_out/r02_attn_ab.json 2>&1
  python -c "
import json,sys
try:
  d=json.loads(open('gpurun_out/r02_attn_ab.json').read().strip().splitlines()[-1]); ob=d['op_breakdown_ms']
  print('$v', round(d['ms_per_step'],3), {k:v for k,v in ob.items() if 'attn' in k or 'softmax' in k or 'flash' in k})
except Exception as e: print('$v failed', open('gpurun_out/r02_attn_ab.json').read()[-800:])"
done
