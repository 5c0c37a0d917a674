#!/bin/sh
# A/B timing of one bench config under env settings (GPU box):
#   tools/ab_config.sh config3 "QG_STAGED=0" "QG_STAGED=1"
CFG=$1; shift
for envs in "$@"; do
  for rep in 1 2; do
    env $envs python bench.py --config $CFG --steps 10 --warmup 3 --no-e2e --no-cpu 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$envs', '$CFG', 'rep$rep', round(d['value']/1e12,2), 'T/s', r['frac'], r['kernel'], d['checksum_c'])"
  done
done
