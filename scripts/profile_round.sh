#!/bin/bash
# Round profile capture on the GPU box (run under gpurun from the repo root):
#   1. a plain bench run (must exit 0 first),
#   2. the launch list of the same command (ncu --metrics gpu__time_duration.sum),
#   3. one `ncu --set full` capture of every kernel of one solve (direct launches).
# Outputs land in gpurun_out/; scripts/profile_summarize.py turns them into profiles/.
set -e
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof_bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/prof_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof_launches.log 2>&1
MFADD_HOST_LOOP=1 ncu --set full --import-source on --clock-control none -k regex:"k_[a-z]" --launch-count 30 \
    -o gpurun_out/prof_full -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e \
    > gpurun_out/prof_full.log 2>&1
ncu -i gpurun_out/prof_full.ncu-rep --page raw --csv > gpurun_out/prof_full_raw.csv
ncu -i gpurun_out/prof_full.ncu-rep --page details > gpurun_out/prof_full_details.txt
rm -f gpurun_out/prof_full.ncu-rep
