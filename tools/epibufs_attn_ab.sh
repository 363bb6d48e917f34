# epilogue staging depth on the epilogue-bound attention GEMMs (score S = QK^T and dP = dO V^T, K = 128)
python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 40 --csv --log-file gpurun_out/ab_base.csv python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
for B in 4 8; do
  MT_NVCC_DEFINES="-DMT_GEMM_EPI_BUFS=$B" python -m paper_2201_11990_b200.build > /dev/null
  ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 40 --csv --log-file gpurun_out/ab_epi$B.csv python bench.py --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
done
