#!/bin/bash
# Collect the round's 1-GPU bench lines (run under gpurun): default + the other configs, logs in gpurun_out/.
mkdir -p gpurun_out
run() {  # name, args...
  local name=$1; shift
  timeout 900 python bench.py "$@" > gpurun_out/rn_$name.json 2> gpurun_out/rn_$name.err
  echo "$name rc=$?"
  grep -h "^{" gpurun_out/rn_$name.json | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if 'roofline' not in d: print(l[:300]); continue
    print(f\"  {d['config']['workload']}: {d['ms_per_step']:.2f} ms, {d.get('tflops_per_gpu',0):.0f} TF/GPU, {d['value']:.0f} tok/s, \"
          f\"gemm {d['roofline']['achieved']:.0f} TF/s ({d['roofline']['frac']:.3f} of sustained), e2e {d['e2e']['value']:.0f}, clocks {d['clocks']['sm_mhz']}\")
"
}
run default --steps 10 --warmup 3
run mtnlg_shard8 --config mtnlg --shard-of 8 --steps 10 --warmup 3 --no-cpu
run mtnlg_shard4 --config mtnlg --shard-of 4 --steps 10 --warmup 3 --no-cpu
run gpt3_shard8 --config gpt3 --shard-of 8 --steps 10 --warmup 3 --no-cpu
run pp1 --config pp --steps 3 --warmup 3 --no-cpu
run tiny --config tiny --steps 10 --warmup 3 --no-cpu
run reference --impl reference --steps 2 --warmup 3
