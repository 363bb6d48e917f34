#!/bin/bash
# Like ab_multi.sh but prints selected ops for every rank. Usage: N=2 OPS="fwd.proj_gemm fwd.fc2_gemm" tools/ab_ranks.sh "ENV1" ...
N=${N:-2}; CFG=${CFG:-gpt3}; port=29700
for cfg in "$@"; do
  port=$((port + 3))
  env $cfg timeout -k 10 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port $port bench.py --gpus $N --steps 5 --warmup 3 --no-cpu --config $CFG --op-timing > gpurun_out/ab.json 2>gpurun_out/ab.err
  grep "^{" gpurun_out/ab.json | tail -1 | OPS="$OPS" python -c "
import json,sys,os
d=json.loads(sys.stdin.read()); b=d['op_breakdown_ms']
print('== $cfg: %.3f ms/step' % d['ms_per_step'])
for op in os.environ['OPS'].split():
    print('   %-28s' % op, '  '.join('%.3f' % b[r].get(op, 0) for r in sorted(b)))
" || tail -5 gpurun_out/ab.err
done
