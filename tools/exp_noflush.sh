show() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().split('\n')[-1]); print(d['roofline']['kernel'], d['roofline']['kernel_ms'], d['roofline']['frac'], round(d['value']/1e12,2), d.get('checksum_c'))"; }
for mode in 0 4; do
for cfg in config5 config2; do
  steps=20; [ $cfg = config5 ] && steps=3
  echo -n "mode $mode $cfg: "; QG_DEBUG_MODE=$mode python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu --no-e2e 2>&1 | show
done; done
