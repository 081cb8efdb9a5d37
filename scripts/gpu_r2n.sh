mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "log_errors or fullsize" 2>&1 | tail -3
for c in C5 C4 C3; do python scripts/time_solve.py --config $c --log-errors --tag ng2; MFADD_RES_NG=1 python scripts/time_solve.py --config $c --log-errors --tag ng1; done
