# The fused backward after removing its register spill: kernel durations (ncu) and the default bench
# step with fused vs unfused attention, alternating.
timeout 600 python -m pytest tests/test_layer_gpu.py -x -q -m gpu 2>&1 | tail -2
python tools/attn_one.py bwd 2 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:attn_ -s 2 -c 4 --csv python tools/attn_one.py bwd 3 2>/dev/null | \
  grep 'gpu__time' | awk -F'","' '{print $5, $NF}' | cut -c1-30,150-
for r in 1 2 3; do
for v in "MT_ATTN_FUSED=0" "MT_ATTN_FUSED=1"; do
  env $v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/ab.json 2>&1
  python -c "
import json
d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
print('$v', round(d['ms_per_step'],3), 'sm', d['clocks']['sm_mhz'], 'loss', round(d['loss'],5))"
done; done
