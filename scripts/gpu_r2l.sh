mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "decode or fullsize or parity or sharded" 2>&1 | tail -3
for kb in 40 24 64; do MFADD_DEC_STAGE_KB=$kb python scripts/time_solve.py --config C4 --tag "kb$kb"; done
python scripts/time_solve.py --config C3 --tag kb40
python scripts/time_solve.py --config C5 --tag c5
MFADD_HOST_LOOP=1 ncu --set full --clock-control none -k regex:"k_decode" -c 1 -o gpurun_out/prof_dec4 -f python scripts/solve_once.py --config C4 > /dev/null 2>&1
ncu -i gpurun_out/prof_dec4.ncu-rep --page raw --csv > gpurun_out/prof_dec4_raw.csv
rm -f gpurun_out/*.ncu-rep
