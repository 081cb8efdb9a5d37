mkdir -p gpurun_out
python scripts/time_solve.py --config C5 --log-errors --tag res2row
python scripts/time_solve.py --config C4 --tag dec_win
python scripts/time_solve.py --config C3 --tag dec_win
MFADD_HOST_LOOP=1 ncu --set full --import-source on --clock-control none -k regex:k_residual -c 1 -o gpurun_out/prof_res -f python scripts/solve_once.py --config C5 --log-errors > /dev/null 2>&1
ncu -i gpurun_out/prof_res.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_res_sass.csv 2>&1
ncu -i gpurun_out/prof_res.ncu-rep --page raw --csv > gpurun_out/prof_res_raw.csv
MFADD_HOST_LOOP=1 ncu --set full --clock-control none -k regex:k_decode -c 1 -o gpurun_out/prof_dec4 -f python scripts/solve_once.py --config C4 > /dev/null 2>&1
ncu -i gpurun_out/prof_dec4.ncu-rep --page raw --csv > gpurun_out/prof_dec4_raw.csv
rm -f gpurun_out/*.ncu-rep
timeout 600 python -m pytest tests -m gpu -x -q -k "decode or fullsize or sharded" 2>&1 | tail -3
