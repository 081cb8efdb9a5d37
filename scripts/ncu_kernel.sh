#!/bin/bash
# ncu --set full (+ source counters) of ONE kernel of a direct-launch solve:
#   bash scripts/ncu_kernel.sh <tag> <kernel regex> <config> [solve_once args]
# -> gpurun_out/k_<tag>_{raw.csv,source.csv}
set -e
tag=$1; k=$2; cfg=$3; shift 3
mkdir -p gpurun_out
MFADD_HOST_LOOP=1 ncu --set full --import-source on --clock-control none -k regex:"$k" --launch-count 1 \
    -o gpurun_out/k_$tag -f python scripts/solve_once.py --config $cfg "$@" > gpurun_out/k_${tag}.log 2>&1
ncu -i gpurun_out/k_$tag.ncu-rep --page raw --csv > gpurun_out/k_${tag}_raw.csv
ncu -i gpurun_out/k_$tag.ncu-rep --page source --csv > gpurun_out/k_${tag}_source.csv 2>/dev/null || true
rm -f gpurun_out/k_$tag.ncu-rep
