#!/bin/bash
# Multi-GPU bench sweep (run under gpurun --gpus N): one bench.py line per config, logs in gpurun_out/.
N=${N:-4}
CFGS=${CFGS:-"gpt3 3d pp mtnlg"}
port=29500
mkdir -p gpurun_out
for cfg in $CFGS; do
  port=$((port + 7))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port $port bench.py --gpus $N --steps ${STEPS:-5} --warmup 3 --config $cfg ${EXTRA:-} \
      > gpurun_out/mb_${cfg}_n$N.json 2> gpurun_out/mb_${cfg}_n$N.err
  echo "$cfg rc=$?"
  python - "$cfg" "$N" <<'PY'
import json, sys
cfg, n = sys.argv[1], sys.argv[2]
try:
    line = [l for l in open(f"gpurun_out/mb_{cfg}_n{n}.json") if l.startswith("{")][-1]
    d = json.loads(line)
    print(f"{d['config']['workload']}: {d['ms_per_step']:.2f} ms, {d['tflops_per_gpu']:.0f} TF/GPU, "
          f"{d['value']:.0f} tok/s, gemm {d['roofline']['achieved']:.0f} TF/s share {d['roofline']['gemm_share_of_step']:.3f}, "
          f"e2e {d['e2e']['value']:.0f}")
except Exception as e:
    print("no result:", e)
    print(open(f"gpurun_out/mb_{cfg}_n{n}.err").read()[-1500:])
PY
done
