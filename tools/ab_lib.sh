#!/bin/bash
# A/B the in-tree libmtnlg.so against _ab_old/paper_2201_11990_b200/libmtnlg.so on the same box (op timing).
OPS=${OPS:-"fwd.attn_s_gemm bwd.attn_dp_gemm fwd.qkv_gemm fwd.fc1_gemm"}
for i in 1 2; do
for t in ${ORDER:-new old}; do
  if [ $t = old ]; then cp paper_2201_11990_b200/libmtnlg.so /tmp/new.so; cp _ab_old/paper_2201_11990_b200/libmtnlg.so paper_2201_11990_b200/libmtnlg.so; fi
  python bench.py --steps 10 --warmup 3 --no-cpu --op-timing $BENCH_ARGS 2>/dev/null | grep "^{" | OPS="$OPS" python -c "
import json,sys,os
d=json.loads(sys.stdin.read()); b=d['op_breakdown_ms']
print('$t', round(d['ms_per_step'],3), round(d['tflops_per_gpu']), {k: b.get(k) for k in os.environ['OPS'].split()})"
  if [ $t = old ]; then cp /tmp/new.so paper_2201_11990_b200/libmtnlg.so; fi
done
done
