# e2e of config 4 / 2 under the 2-D host pipeline: panels x tiles-per-launch
show() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().split('\n')[-1]); e=d.get('e2e',{}); print(round(e.get('value',0)/1e12,2), 'T/s e2e', round(e.get('ms_per_step',0),3), 'ms')"; }
for cfg in config4 config2; do
  for P in 2 4; do
    for T in 48 96 192; do
      echo -n "$cfg P=$P T=$T: "; QG_HOST_PANELS=$P QG_HOST_TILES=$T python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu --e2e-steps 3 2>&1 | show
    done
  done
done
