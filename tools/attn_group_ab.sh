# Launch-order grouping of the fused attention kernels (MT_ATTN_GROUP_HEADS heads per group, 0 = all
# heads in one group): ncu duration and DRAM bytes, GPT-3 layer shape.
for r in 1 2; do
for g in 0 4 8 12; do
  MT_ATTN_GROUP_HEADS=$g python tools/attn_one.py bwd 2 > /dev/null 2>&1
  MT_ATTN_GROUP_HEADS=$g ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"attn_fwd2|attn_bwd2" -s 2 -c 2 --csv python tools/attn_one.py bwd 2 2>/dev/null | \
    grep -E 'gpu__time|dram__bytes' | awk -F'","' -v c="group=$g" '{print c, substr($5,1,30), $(NF-2), $NF}'
done; done
