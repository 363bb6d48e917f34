# Reducer CTAs of the fused GEMM + NVLS all-reduce (MT_AR_CTAS, default 16) at N=4, alternating.
port=29900
for r in 1 2 3; do
for CFG in gpt3 mtnlg; do
for v in 16 24 32; do
  port=$((port + 3))
  MT_AR_CTAS=$v timeout -k 10 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
      --master-port $port bench.py --gpus 4 --steps 10 --warmup 3 --no-cpu --config $CFG 2>/dev/null | grep "^{" | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$CFG MT_AR_CTAS=$v', round(d['ms_per_step'],3), round(d['roofline']['achieved']))"
done; done; done
