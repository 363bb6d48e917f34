# dK/dV + dQ kernel pair (hd 160 default fused backward; hd 128 with MT_ATTN_BWD2=0) with one vs two
# softmax warpgroups: ncu durations.
for wg in 1 2; do
for cfg in "H=2560 HEADS=16" "H=12288 HEADS=96 MT_ATTN_BWD2=0"; do
  env $cfg MT_ATTN_BWD_WG=$wg python tools/attn_one.py bwd 2 > /dev/null 2>&1
  env $cfg MT_ATTN_BWD_WG=$wg ncu --metrics gpu__time_duration.sum --clock-control none -k regex:attn_bwd_d -s 2 -c 2 --csv python tools/attn_one.py bwd 3 2>/dev/null | \
    grep 'gpu__time' | awk -F'","' -v c="WG=$wg $cfg" '{print c, substr($5,1,40), $NF}'
done; done
