# mbarrier try_wait with a suspend-time hint (new) vs plain polling (old, _ab_old): ncu durations of the
# attention and row kernels and of the GEMMs of one default step, then the bench step, alternating.
for t in new old; do
  if [ $t = old ]; then d=_ab_old; else d=.; fi
  (cd $d && python tools/attn_one.py bwd 2 > /dev/null 2>&1 && \
   ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attn_fwd2|attn_bwd2" -s 2 -c 2 --csv python tools/attn_one.py bwd 3 2>/dev/null | \
     grep gpu__time | awk -F'","' -v c=$t '{print c, substr($5,1,40), $NF}')
  (cd $d && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"_rows_kernel|gemm_sm100" -s 20 -c 20 --csv \
     python bench.py --steps 1 --warmup 1 --no-cpu 2>/dev/null | grep gpu__time | awk -F'","' -v c=$t '{s+=$NF; if ($5 ~ /rows/) r+=$NF; else g+=$NF} END {print c, "rows_us", r/1000, "gemm_us", g/1000}')
done
for r in 1 2 3; do
for t in new old; do
  if [ $t = old ]; then d=_ab_old; else d=.; fi
  (cd $d && python bench.py --steps 20 --warmup 5 --no-cpu 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$t', round(d['ms_per_step'],3), 'sm', d['clocks']['sm_mhz'])")
done; done
