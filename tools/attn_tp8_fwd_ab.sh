# GPT-3 TP=8 shard attention (12 local heads): two-tile forward (96 CTAs) vs single-tile (192 CTAs)
for v in 1 0; do
  H=1536 HEADS=12 MT_ATTN_FWD2=$v python tools/attn_one.py bwd 2 > /dev/null 2>&1
  H=1536 HEADS=12 MT_ATTN_FWD2=$v ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attn_" -s 4 -c 4 --csv python tools/attn_one.py bwd 3 2>/dev/null | \
    grep gpu__time | awk -F'","' -v c="fwd2=$v" '{print c, substr($5,1,40), $NF}'
done
