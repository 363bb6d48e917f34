# Attention kernel durations (ncu) at the GPT-3 shape (hd 128) and the MT-NLG TP=8 shard shape (hd 160,
# forced fused) — run on the tree under test.
for cfg in "H=12288 HEADS=96" "H=2560 HEADS=16"; do
  env $cfg python tools/attn_one.py bwd 2 > /dev/null 2>&1
  env $cfg ncu --metrics gpu__time_duration.sum --clock-control none -k regex:attn_ -s 4 -c 4 --csv python tools/attn_one.py bwd 3 2>/dev/null | \
    grep 'gpu__time' | awk -F'","' -v c="$cfg" '{print c, substr($5,1,40), $NF}'
done
