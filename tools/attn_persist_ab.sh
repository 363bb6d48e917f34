# Persistent one-kernel attention backward (one CTA per SM walking the work items) vs one CTA per
# item: ncu durations at the GPT-3 shape and across sequence lengths.
for r in 1 2; do
for v in 1 0; do
for cfg in "H=12288 HEADS=96 SEQ=2048" "H=6144 HEADS=48 SEQ=4096" "H=12288 HEADS=96 SEQ=1024"; do
  env $cfg MT_ATTN_PERSIST=$v python tools/attn_one.py bwd 2 > /dev/null 2>&1
  env $cfg MT_ATTN_PERSIST=$v ncu --metrics gpu__time_duration.sum --clock-control none -k regex:attn_bwd2 -s 1 -c 1 --csv python tools/attn_one.py bwd 2 2>/dev/null | \
    grep 'gpu__time' | awk -F'","' -v c="persist=$v $cfg" '{print c, substr($5,1,40), $NF}'
done; done; done
