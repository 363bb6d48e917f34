# Two-tile forward pairing: adjacent query blocks vs balanced (heavy + light) pairs, at the GPT-3 TP=8
# (12 heads), TP=4 (24), TP=2 (48) and TP=1 (96) shard shapes.
for heads in 12 24 48 96; do
for v in 0 1; do
  H=$((heads * 128)) HEADS=$heads MT_ATTN_FWD_BALANCED=$v python tools/attn_one.py fwd 2 > /dev/null 2>&1
  H=$((heads * 128)) HEADS=$heads MT_ATTN_FWD_BALANCED=$v ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attn_fwd2" -s 1 -c 1 --csv python tools/attn_one.py fwd 2 2>/dev/null | \
    grep gpu__time | awk -F'","' -v c="heads=$heads balanced=$v" '{print c, $NF}'
done; done
