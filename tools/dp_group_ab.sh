# A/B (run under gpurun --gpus 2): the DP gradient all-reduce per parameter group during the last
# backward (default) vs per layer after its backward (MT_DP_PER_GROUP=0), config dp (DP=2, h=8192 x 2 layers, MB=4).
port=29600
for r in 1 2; do
  for g in 0 1; do
    port=$((port + 3))
    MT_DP_PER_GROUP=$g timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
      --master-port $port bench.py --gpus 2 --steps 10 --warmup 3 --config dp --no-cpu 2> gpurun_out/dpg_$g.err | \
      python -c "import json,sys; d=json.loads([l for l in sys.stdin.read().splitlines() if l.startswith('{')][-1]); print('per_group=$g', round(d['ms_per_step'],2), round(d['tflops_per_gpu']), d['clocks']['sm_mhz'], d['clocks'].get('power_w_max'))"
  done
done
