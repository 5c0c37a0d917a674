#!/bin/sh
# DRAM bytes + duration of the first K4 launch of a config under env settings
# (GPU box): tools/ab_ncu_dram.sh config5 "QG_GROUP=8" "QG_GROUP=16"
CFG=$1; shift
mkdir -p gpurun_out
for envs in "$@"; do
  tag=$(echo "$envs" | tr ' =' '__')
  env $envs ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
      --clock-control none -k regex:k_gemm_tiled -c 1 --csv \
      python bench.py --config $CFG --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/dram_${CFG}_$tag.csv 2>&1
done
