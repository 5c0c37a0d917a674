# config-4 e2e: k-split host path (default for this shape) vs the 1-D pipeline
show() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().split('\n')[-1]); e=d.get('e2e',{}); print(round(e.get('value',0)/1e12,2), 'T/s e2e', round(e.get('ms_per_step',0),3), 'ms', d.get('cc_sha256'))"; }
for v in 1 0; do
  for P in 4 8 16; do
    echo -n "ksplit=$v parts=$P config4: "; QG_HOST_KSPLIT=$v QG_HOST_KPARTS=$P python bench.py --config config4 --steps 2 --warmup 3 --no-cpu 2>&1 | show
    [ $v = 0 ] && break
  done
done
