#!/bin/bash
# A/B env variants for a multi-GPU bench (op breakdown of rank 0). Usage: N=4 tools/ab_multi.sh "ENV1" "ENV2" ...
N=${N:-4}; CFG=${CFG:-gpt3}; port=29600
for cfg in "$@"; do
  port=$((port + 3))
  env $cfg timeout -k 10 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port $port bench.py --gpus $N --steps 5 --warmup 3 --no-cpu --config $CFG --op-timing > gpurun_out/ab.json 2>gpurun_out/ab.err
  grep "^{" gpurun_out/ab.json | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); b=d['op_breakdown_ms']['rank0']
print('== $cfg: %.3f ms/step, %.0f TF/GPU' % (d['ms_per_step'], d['tflops_per_gpu']))
print('   ' + ', '.join('%s %.3f' % kv for kv in sorted(b.items(), key=lambda kv: -kv[1])[:10]))
" || tail -5 gpurun_out/ab.err
done
