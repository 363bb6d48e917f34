# attention row term D = rowsum(dO * O): coalesced vector kernel (new) vs warp-per-row (hd 160 path)
for cfg in "H=12288 HEADS=96" "H=2560 HEADS=16"; do
  env $cfg python tools/attn_one.py bwd 2 > /dev/null 2>&1
  env $cfg ncu --metrics gpu__time_duration.sum --clock-control none -k regex:rowdot -c 2 --csv python tools/attn_one.py bwd 2 2>/dev/null | \
    grep 'gpu__time' | awk -F'","' -v c="$cfg" '{print c, substr($5,1,50), $NF}'
done
