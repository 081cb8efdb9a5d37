mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "parity or golden or fullsize or shim or sharded or boundary" 2>&1 | tail -3
for c in C5 C2; do python scripts/time_solve.py --config $c --tag split; MFADD_SOLVE2D=1 python scripts/time_solve.py --config $c --tag cta; done
MFADD_HOST_LOOP=1 ncu --set full --clock-control none -k regex:"k_rows2d|k_cols2d|k_last_contract" -c 3 -o gpurun_out/prof_split -f python scripts/solve_once.py --config C5 > /dev/null 2>&1
ncu -i gpurun_out/prof_split.ncu-rep --page raw --csv > gpurun_out/prof_split_raw.csv
rm -f gpurun_out/*.ncu-rep
