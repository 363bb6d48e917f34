for cfg in "H=12288 HEADS=96 SEQ=2048" "H=6144 HEADS=48 SEQ=4096" "H=12288 HEADS=96 SEQ=1024"; do
  env $cfg python tools/attn_one.py bwd 2 > /dev/null 2>&1
  env $cfg ncu --metrics gpu__time_duration.sum --clock-control none -k regex:attn_ -s 2 -c 2 --csv python tools/attn_one.py bwd 3 2>/dev/null | \
    grep 'gpu__time' | awk -F'","' -v c="$cfg" '{print c, substr($5,1,40), $NF}'
done
