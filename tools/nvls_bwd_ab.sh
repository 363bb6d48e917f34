#!/bin/bash
# Backward "f" all-reduces: NCCL on the 16-CTA side communicator vs the NVLS kernel (bwd CTAs 16 / 8),
# N=4 TP=4 GPT-3 and MT-NLG layers, alternating; ms/step of the max over ranks.
N=${N:-4}; port=29700
for r in 1 2; do
for CFG in gpt3 mtnlg; do
for v in "MT_TP_NVLS_BWD=0" "MT_TP_NVLS_BWD=1" "MT_TP_NVLS_BWD=1 MT_NVLS_BWD_CTAS=8"; do
  port=$((port + 3))
  env $v timeout -k 10 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port $port bench.py --gpus $N --steps 10 --warmup 3 --no-cpu --config $CFG > gpurun_out/ab.json 2>gpurun_out/ab.err
  grep "^{" gpurun_out/ab.json | tail -1 | V="$v" C=$CFG python -c "
import json,sys,os
d=json.loads(sys.stdin.read())
print(os.environ['C'], os.environ['V'], '%.3f ms/step %.0f TF/GPU sm %s' % (d['ms_per_step'], d['tflops_per_gpu'], d['clocks'].get('sm_mhz')))" || tail -5 gpurun_out/ab.err
done; done; done
