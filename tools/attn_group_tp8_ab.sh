# Backward launch-order grouping at the TP=8 (12 heads) and TP=4 (24 heads) GPT-3 shard shapes
for heads in ${HEADS_LIST:-12 24}; do
for g in 0 4 8; do
  H=$((heads * 128)) HEADS=$heads MT_ATTN_GROUP_HEADS=$g python tools/attn_one.py bwd 2 > /dev/null 2>&1
  H=$((heads * 128)) HEADS=$heads MT_ATTN_GROUP_HEADS=$g ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attn_bwd2" -s 1 -c 1 --csv python tools/attn_one.py bwd 2 2>/dev/null | \
    grep gpu__time | awk -F'","' -v c="heads=$heads group=$g" '{print c, $NF}'
done; done
