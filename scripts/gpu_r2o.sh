mkdir -p gpurun_out
for c in C4 C3; do python scripts/time_solve.py --config $c --tag morton; MFADD_NO_MORTON=1 python scripts/time_solve.py --config $c --tag lex; done
timeout 600 python -m pytest tests -m gpu -x -q -k "C3s or C4s or fullsize or 3d" 2>&1 | tail -2
MFADD_HOST_LOOP=1 ncu --set full --clock-control none -k regex:"k_fit_axis0" -c 2 -o gpurun_out/prof_ax0 -f python scripts/solve_once.py --config C4 > /dev/null 2>&1
ncu -i gpurun_out/prof_ax0.ncu-rep --page raw --csv > gpurun_out/prof_ax0_raw.csv
rm -f gpurun_out/*.ncu-rep
