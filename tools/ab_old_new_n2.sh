# Same-box A/B of the in-tree library vs _ab_old at N=2 (GPT-3 layer TP=2), alternating.
port=29811
for r in 1 2 3; do
for t in new old; do
  if [ $t = old ]; then d=_ab_old; else d=.; fi
  port=$((port + 3))
  (cd $d && timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
     --master-port $port bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu 2>/dev/null | grep "^{" | tail -1 | \
     python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$t', round(d['ms_per_step'],3), round(d['roofline']['achieved']))")
done; done
