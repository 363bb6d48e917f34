# Per-op breakdown of one TP=8 shard (compute only) for the MT-NLG and GPT-3 layers.
for cfg in "--config mtnlg --shard-of 8" "--config gpt3 --shard-of 8"; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --op-timing $cfg 2>/dev/null | grep "^{" | C="$cfg" python -c "
import json,sys,os
d=json.loads(sys.stdin.read()); b=d['op_breakdown_ms']
print('==', os.environ['C'], round(d['ms_per_step'],3), 'ms', 'sm', d['clocks'].get('sm_mhz'))
print('   ' + ', '.join('%s %.3f' % kv for kv in sorted(b.items(), key=lambda kv: -kv[1])))"
done
