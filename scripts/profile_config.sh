#!/bin/bash
# ncu --set full of every kernel of one direct-launch solve of a config
#   bash scripts/profile_config.sh C4 [--log-errors]   -> gpurun_out/prof_<tag>_{raw.csv,details.txt}
set -e
cfg=$1; shift
tag=$cfg
if [ "$1" = "--log-errors" ]; then tag=${cfg}_le; fi
mkdir -p gpurun_out
python scripts/solve_once.py --config $cfg "$@" > gpurun_out/prof_${tag}_plain.log 2>&1
MFADD_HOST_LOOP=1 ncu --set full --import-source on --clock-control none -k regex:"${NCU_K:-k_[a-z]}" --launch-count ${NCU_COUNT:-40} \
    -o gpurun_out/prof_$tag -f python scripts/solve_once.py --config $cfg "$@" > gpurun_out/prof_${tag}.log 2>&1
ncu -i gpurun_out/prof_$tag.ncu-rep --page raw --csv > gpurun_out/prof_${tag}_raw.csv
ncu -i gpurun_out/prof_$tag.ncu-rep --page details > gpurun_out/prof_${tag}_details.txt
[ -n "$NCU_SOURCE" ] && ncu -i gpurun_out/prof_$tag.ncu-rep --page source --csv > gpurun_out/prof_${tag}_source.csv 2>/dev/null || true
rm -f gpurun_out/prof_$tag.ncu-rep
