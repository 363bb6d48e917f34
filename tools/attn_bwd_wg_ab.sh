# One-kernel attention backward with one vs two softmax warpgroups (column halves): ncu kernel
# durations (ns) of the fused attention kernels, alternating.
for r in 1 2; do
for wg in 1 2; do
  MT_ATTN_BWD_WG=$wg python tools/attn_one.py bwd 2 > /dev/null 2>&1
  MT_ATTN_BWD_WG=$wg ncu --metrics gpu__time_duration.sum --clock-control none -k regex:attn_ -s 2 -c 4 --csv python tools/attn_one.py bwd 3 2>/dev/null | \
    grep 'gpu__time' | awk -F'","' -v wg=$wg '{print "WG=" wg, substr($5,1,40), $NF}'
done; done
