#!/bin/bash
# Full rank-0 op breakdown side by side for env variants. Usage: N=4 tools/ab_full.sh "ENV1" "ENV2"
N=${N:-4}; CFG=${CFG:-gpt3}; port=29800; i=0
for cfg in "$@"; do
  port=$((port + 3)); i=$((i+1))
  env $cfg timeout -k 10 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port $port bench.py --gpus $N --steps 5 --warmup 3 --no-cpu --config $CFG --op-timing > gpurun_out/abf_$i.json 2>/dev/null
done
python - "$@" <<'PY'
import json, sys
ds = []
for i in range(1, len(sys.argv)):
    line = [l for l in open(f"gpurun_out/abf_{i}.json") if l.startswith("{")][-1]
    ds.append(json.loads(line))
print("ms/step", [round(d["ms_per_step"], 3) for d in ds])
keys = sorted(set().union(*[d["op_breakdown_ms"]["rank0"] for d in ds]), key=lambda k: -ds[0]["op_breakdown_ms"]["rank0"].get(k, 0))
for k in keys:
    print("%-34s" % k, "  ".join("%.3f" % d["op_breakdown_ms"]["rank0"].get(k, 0) for d in ds))
PY
