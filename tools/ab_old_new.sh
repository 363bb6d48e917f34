for i in 1 2; do
for t in new old; do
  if [ $t = old ]; then d=_ab_old; else d=.; fi
  (cd $d && python bench.py --steps 10 --warmup 3 --no-cpu 2>/dev/null | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$t', round(d['ms_per_step'],3), round(d['tflops_per_gpu']), round(d['roofline']['achieved']), d['clocks']['sm_mhz'])")
done
done
