# config-4 right/left variant: planner pick vs alternative (t, e, k-block, balanced) plans
show() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().split('\n')[-1]); print(round(d['ms_per_step'],3), d['roofline']['kernel_ms'], d['roofline']['frac'], round(d['value']/1e12,1), d['checksum_c'], d['config']['plan'])"; }
echo -n "planner: "; python bench.py --config config4 --steps 10 --warmup 3 --no-cpu --no-e2e 2>&1 | show
for pl in 13:4:504:0 13:4:1008:1 13:4:504:1 12:4:504:1 10:5:112:1 10:5:56:0; do
  echo -n "$pl: "; python bench.py --config config4 --steps 10 --warmup 3 --no-cpu --no-e2e --redq-plan $pl 2>&1 | show
done
echo -n "left planner: "; python bench.py --config config4_left --steps 10 --warmup 3 --no-cpu --no-e2e 2>&1 | show
echo -n "left 13:4:1008:1: "; python bench.py --config config4_left --steps 10 --warmup 3 --no-cpu --no-e2e --redq-plan 13:4:1008:1 2>&1 | show
