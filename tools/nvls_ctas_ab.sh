# standalone NVLS all-reduce CTA count: probe + TP=N layer bench (run under gpurun --gpus N)
N=${N:-4}
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29621 tools/nvls_probe.py 2>&1 | grep "TP="
port=29630
for rep in 1 2; do
for c in 16 32 64 148; do
  port=$((port+1))
  MT_NVLS_CTAS=$c timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $port bench.py --gpus $N --steps 10 --warmup 3 --no-cpu --op-timing 2>/dev/null | grep "^{" | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); o=d['op_breakdown_ms']['rank0']; print('ctas=$c', round(d['ms_per_step'],3), 'fwd.tp_allreduce', o.get('fwd.tp_allreduce'), 'fc2', o.get('fwd.fc2_gemm'), d['clocks']['sm_mhz'])"
done
done
