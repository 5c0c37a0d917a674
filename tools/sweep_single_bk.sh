# single-block stage depth sweep (config 3 by default)
for bk in 52 44 36 28 20 12; do
  echo "== BK=$bk"; QG_TILED_SINGLE_BK=$bk python bench.py --config ${CFG:-config3} --steps 20 --warmup 5 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), d['roofline']['kernel_ms'], d['roofline']['frac'], round(d['value']/1e12,2), d['checksum_c'] if 'checksum_c' in d else '')"
done
