# K4 warp-skew sweep on configs 2 and 5 under the current flush scheme
show() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().split('\n')[-1]); print(d['roofline']['kernel_ms'], d['roofline']['frac'], d['checksum_rank0'])"; }
for sk in 0 2000 4000 6000 10000; do
  for cfg in config2 config5; do
    steps=20; [ $cfg = config5 ] && steps=2
    echo -n "skew=$sk $cfg: "; QG_SKEW_NS=$sk python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu --no-e2e 2>&1 | show
  done
done
