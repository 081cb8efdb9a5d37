mkdir -p gpurun_out
for i in 1 2; do python scripts/time_solve.py --config C5 --tag lines2; MFADD_SOLVE2D_LINES=1 python scripts/time_solve.py --config C5 --tag lines1; done
python scripts/time_solve.py --config C2 --tag lines2; MFADD_SOLVE2D_LINES=1 python scripts/time_solve.py --config C2 --tag lines1
timeout 600 python -m pytest tests -m gpu -x -q -k "parity or golden or shim" 2>&1 | tail -2
MFADD_HOST_LOOP=1 ncu --set full --clock-control none -k regex:"k_solve2d" -c 1 -o gpurun_out/prof_s2d -f python scripts/solve_once.py --config C5 > /dev/null 2>&1
ncu -i gpurun_out/prof_s2d.ncu-rep --page raw --csv > gpurun_out/prof_s2d_raw.csv
rm -f gpurun_out/*.ncu-rep
