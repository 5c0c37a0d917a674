show() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().split('\n')[-1]); print(round(d['ms_per_step'],4), d['roofline']['kernel_ms'], d['roofline']['frac'], round(d['value']/1e12,2), d['config']['plan']['stage_words'], d['gpu_launches'], d['checksum_rank0'], d['config'].get('launch'))"; }
for c in config1 config3 config2; do
  echo "== $c graph"; python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-e2e 2>&1 | show
  echo "== $c no-graph"; python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-e2e --no-graph 2>&1 | show
done
echo "== config2 reference plan (auto bk)"; python bench.py --config config2 --plan reference --steps 10 --warmup 3 --no-cpu --no-e2e 2>&1 | show
echo "== config2 reference plan bk28"; QG_TILED_SINGLE_BK=28 python bench.py --config config2 --plan reference --steps 10 --warmup 3 --no-cpu --no-e2e 2>&1 | show
