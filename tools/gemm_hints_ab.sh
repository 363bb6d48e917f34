# L2 eviction-hint modes on the m-fastest forward GEMM (fc1 fwd, GPT-3 TP=1): time + DRAM bytes
for h in 0 1 2; do
  MT_GEMM_HINTS=$h python tools/gemm_one.py ${G:-fc1_fwd} 6 | tail -2
  MT_GEMM_HINTS=$h ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gemm_sm100 -s 3 -c 1 python tools/gemm_one.py ${G:-fc1_fwd} 4 2>/dev/null | grep -E "dram__bytes|duration" | sed "s/^/hints=$h /"
done
