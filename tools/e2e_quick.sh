# e2e (host buffers through the public API): the library's pipeline choice
# (QG_HOST_2D unset) against forcing the 2-D (1) or 1-D (0) host pipeline
show() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().split('\n')[-1]); e=d.get('e2e',{}); print(round(e.get('value',0)/1e12,2), 'T/s e2e', round(e.get('ms_per_step',0),3), 'ms', e.get('checksum_rank0', e.get('cc_sha256')))"; }
for v in auto 1 0; do
  if [ $v = auto ]; then unset QG_HOST_2D; else export QG_HOST_2D=$v; fi
  for cfg in config2 config4; do
    echo -n "2d=$v $cfg: "; python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu 2>&1 | show
  done
  echo -n "2d=$v config5: "; python bench.py --config config5 --steps 1 --warmup 3 --no-cpu --e2e-steps 2 2>&1 | show
done
