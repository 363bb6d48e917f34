# e2e (host-input) step time vs the number of row chunks the first layer consumes the input in
for r in 1 2; do
for k in 4 8 2; do
  MT_INPUT_CHUNKS=$k timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/ab.json 2>&1
  python -c "
import json
d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
print('chunks $k', 'dev', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],3), 'gap', round(d['e2e']['ms_per_step']-d['ms_per_step'],3), 'sm', d['clocks']['sm_mhz'])"
done; done
