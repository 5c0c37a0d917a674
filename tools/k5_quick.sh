# Quick K5 check (tiled mixed / left / full variants on config 4's shape)
show() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().split('\n')[-1]); print(d['roofline']['kernel'], d['roofline']['kernel_ms'], d['roofline']['frac'], round(d['value']/1e12,2), d.get('cc_sha256', d.get('checksum_rank0')))"; }
for cfg in config4 config4_left config4_full; do
  echo -n "$cfg: "; python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-e2e 2>&1 | show
done
