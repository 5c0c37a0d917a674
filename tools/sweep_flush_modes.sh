# K4 flush mode / skew sweep on configs 2 and 5 (proxy rows for 5)
show() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().split('\n')[-1]); print(d['roofline']['kernel_ms'], d['roofline']['frac'], d['checksum_rank0'])"; }
for cfg in config2 config5; do
  steps=10; [ $cfg = config5 ] && steps=2
  for f in 3 0 1; do
    for sk in 4000 8000; do
      echo -n "$cfg flush=$f skew=$sk: "; QG_FLUSH=$f QG_SKEW_NS=$sk python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu --no-e2e 2>&1 | show
    done
  done
done
