#!/bin/sh
# ncu --set full capture of one contraction launch of tools/k4_micro.py; CSV summaries only travel back.
# usage: tools/ncu_micro.sh <name> <kernel regex> [k4_micro args]
set -e
NAME=$1; KRE=$2; shift; shift
OUT=gpurun_out/ncu_$NAME
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:$KRE -s 2 -c 1 -o $OUT python tools/k4_micro.py --reps 1 "$@" > $OUT.log 2>&1
ncu -i $OUT.ncu-rep --page raw --csv > ${OUT}_raw.csv
ncu -i $OUT.ncu-rep --page source --csv --print-source sass > ${OUT}_sass.csv 2>/dev/null || true
gzip -f ${OUT}_sass.csv
rm -f $OUT.ncu-rep
