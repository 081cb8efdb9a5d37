mkdir -p gpurun_out
for kb in 24 16; do MFADD_DEC_STAGE_KB=$kb python scripts/time_solve.py --config C4 --tag "kb$kb"; done
MFADD_HOST_LOOP=1 python scripts/time_solve.py --config C5 --tag hostloop
MFADD_HOST_LOOP=1 ncu --set full --clock-control none -k regex:"k_[a-z]" -c 40 -o gpurun_out/prof_C4all -f python scripts/solve_once.py --config C4 > /dev/null 2>&1
ncu -i gpurun_out/prof_C4all.ncu-rep --page raw --csv > gpurun_out/prof_C4all_raw.csv
rm -f gpurun_out/*.ncu-rep
