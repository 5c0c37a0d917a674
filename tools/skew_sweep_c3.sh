# warp-skew sweep for the single-block tiles of config 3
show() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().split('\n')[-1]); print(d['roofline']['kernel_ms'], d['roofline']['frac'], d['checksum_rank0'])"; }
for sk in 0 2000 3000 4000 5000 6000 8000; do
  echo -n "skew=$sk config3: "; QG_SKEW_NS=$sk python bench.py --config config3 --steps 20 --warmup 3 --no-cpu --no-e2e 2>&1 | show
done
