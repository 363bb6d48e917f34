#!/bin/bash
# ncu evidence (run under gpurun, 1 GPU). Every profiled command first exits 0 without ncu.
#   1. per-launch durations of the bench command (cold-cache, serialised: compare SHARES)
#   2. --set full on representative tcgen05 GEMMs (fwd K-major, dgrad MN-major B, wgrad MN x MN fp32)
#   3. --set full on the HBM-bound kernels of one bench step
set -e
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu"
$CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD \
    > gpurun_out/ncu_launches.log 2>&1
for g in ${GEMMS:-fc1_fwd fc1_dgrad fc1_wgrad}; do
  python tools/gemm_one.py $g 3 > gpurun_out/gemm_$g.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:gemm_sm100 -s 2 -c 1 \
      -o gpurun_out/prof_gemm_$g python tools/gemm_one.py $g 3 > gpurun_out/ncu_gemm_$g.log 2>&1
done
ncu --set full --clock-control none -k regex:"softmax|ln_|colsum|bias_dropout|bdr_|rows_kernel|mse" -s 12 -c ${HBM_COUNT:-12} \
    -o gpurun_out/prof_hbm $CMD > gpurun_out/ncu_hbm.log 2>&1
echo done
