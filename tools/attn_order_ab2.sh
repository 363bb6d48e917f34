# Old (head-major launch order) vs new (heavy-first across heads) attention kernels, ncu durations.
for r in 1 2; do
for t in new old; do
  if [ $t = old ]; then d=_ab_old; else d=.; fi
  (cd $d && MT_ATTN_FUSED=1 bash tools/attn_order_ab.sh | sed "s/^/$t /")
done; done
