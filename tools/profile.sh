#!/bin/bash
# ncu evidence for the bench command (run under gpurun, 1 GPU). Plain run first (must exit 0),
# then the per-launch duration list, then one full capture of the top GEMM launches.
set -e
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu"
$CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD \
    > gpurun_out/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_sm100 -s 30 -c 4 \
    -o gpurun_out/prof_gemm $CMD > gpurun_out/ncu_full.log 2>&1
ncu --set full --clock-control none -k regex:"softmax|ln_|colsum|bias_dropout" -s 6 -c 8 \
    -o gpurun_out/prof_hbm $CMD > gpurun_out/ncu_hbm.log 2>&1
echo done
