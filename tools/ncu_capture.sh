#!/bin/sh
# ncu --set full capture of the first K4 launch of a bench config, exported on
# the box to CSV (raw metrics + per-source-line stalls) so only the summaries
# travel back. Usage (on the GPU box): tools/ncu_capture.sh config5 [extra bench args]
set -e
CFG=$1; shift
OUT=gpurun_out/ncu_$CFG
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:k_gemm_ -c 1 -o $OUT \
    python bench.py --config $CFG --steps 1 --warmup 3 --no-e2e --no-cpu "$@" > $OUT.log 2>&1
ncu -i $OUT.ncu-rep --page raw --csv > ${OUT}_raw.csv
ncu -i $OUT.ncu-rep --page source --csv --print-source sass > ${OUT}_sass.csv 2>/dev/null || true
ncu -i $OUT.ncu-rep --page details --csv > ${OUT}_details.csv
gzip -f ${OUT}_sass.csv
rm -f $OUT.ncu-rep
