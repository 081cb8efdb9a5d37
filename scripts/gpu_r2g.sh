mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "log_errors" 2>&1 | tail -3
for c in C5 C4 C3 C2; do python scripts/time_solve.py --config $c --log-errors --tag dense; MFADD_RES_ROWS=1 python scripts/time_solve.py --config $c --log-errors --tag rows; done
MFADD_HOST_LOOP=1 ncu --set full --import-source on --clock-control none -k regex:k_residual -c 1 -o gpurun_out/prof_res -f python scripts/solve_once.py --config C5 --log-errors > /dev/null 2>&1
ncu -i gpurun_out/prof_res.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_res_sass.csv 2>&1
ncu -i gpurun_out/prof_res.ncu-rep --page raw --csv > gpurun_out/prof_res_raw.csv
rm -f gpurun_out/*.ncu-rep
