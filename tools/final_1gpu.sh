#!/bin/bash
# Round-end evidence on one B200 (run under gpurun): GPU suite, smoke, default bench + CPU reference arm,
# compute-only TP shard benches, launch list of the default bench, ncu --set full of the dominant GEMM.
set -u
mkdir -p gpurun_out
R=${R:-r02}
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=8 > gpurun_out/${R}_final_gpu1.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${R}_final_gpu1.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${R}_final_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${R}_final_smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/${R}_bench_default.json 2> gpurun_out/${R}_bench_default.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${R}_bench_reference.json 2>&1; echo "ref rc=$?"
for a in "--config mtnlg --shard-of 8" "--config gpt3 --shard-of 8" "--config mtnlg --shard-of 4" "--config gpt3 --recompute"; do
  n=$(echo $a | tr -d ' -' )
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu $a > gpurun_out/${R}_bench_$n.json 2>&1; echo "$a rc=$?"
done
python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/${R}_launches_final.csv \
      python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1; echo "ncu launches rc=$?"
python tools/gemm_one.py fc1_fwd 3 > /dev/null 2>&1 && \
  ncu --set full --import-source on --clock-control none -k regex:gemm_sm100 -s 2 -c 1 -o gpurun_out/${R}_gemm_fc1_fwd \
      python tools/gemm_one.py fc1_fwd 3 > /dev/null 2>&1; echo "ncu gemm rc=$?"
for f in gpurun_out/${R}_bench_*.json; do echo "== $f"; tail -c 600 $f; echo; done
# fused attention kernels of the default path (GPT-3 layer shape), full section set
python tools/attn_one.py bwd 2 > /dev/null 2>&1 && \
  ncu --set full --import-source on --clock-control none -k regex:"attn_fwd2|attn_bwd2" -s 2 -c 2 -o gpurun_out/${R}_attn_final \
      python tools/attn_one.py bwd 3 > /dev/null 2>&1; echo "ncu attn rc=$?"
