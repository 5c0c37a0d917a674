# Quick K4 check: contraction time / roofline fraction / checksum for configs 2, 3, 5
show() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().split('\n')[-1]); print(d['roofline']['kernel'], d['roofline']['kernel_ms'], d['roofline']['frac'], round(d['value']/1e12,2), d['checksum_rank0'])"; }
for cfg in config2 config3 config5; do
  steps=20; [ $cfg = config5 ] && steps=3
  echo -n "$cfg: "; python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu --no-e2e 2>&1 | show
done
