#!/bin/bash
# Where the TP communication goes at N=4: op breakdown of one TP=4 shard computed alone (--shard-of 4,
# no collectives) vs the real TP=4 run (default fused/NVLS paths) vs reducer-CTA and fused-off variants.
port=29800
show() { python -c "
import json,sys
t=[l for l in open('$1').read().splitlines() if l.startswith('{')]
d=json.loads(t[-1]); b=d.get('op_breakdown_ms',{}); b=b.get('rank0',b)
print('== $2: %.3f ms/step, %.0f TF/GPU' % (d['ms_per_step'], d['tflops_per_gpu']))
print('   ' + ', '.join('%s %.3f' % kv for kv in sorted(b.items(), key=lambda kv: -kv[1])[:16]))
" || tail -3 $1; }
for CFG in mtnlg gpt3; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --config $CFG --shard-of 4 --op-timing > gpurun_out/s.json 2>&1
  show gpurun_out/s.json "$CFG shard-of-4 (compute only)"
  for v in "MT_TP_FUSED=1" "MT_TP_FUSED=1 MT_AR_CTAS=32" "MT_TP_FUSED=0 MT_TP_NVLS=1"; do
    port=$((port + 3))
    env $v timeout -k 10 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
      --master-port $port bench.py --gpus 4 --steps 10 --warmup 3 --no-cpu --config $CFG --op-timing > gpurun_out/m.json 2>gpurun_out/m.err
    show gpurun_out/m.json "$CFG N=4 $v"
  done
done
