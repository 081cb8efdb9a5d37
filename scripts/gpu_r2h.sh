mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "log_errors" 2>&1 | tail -3
for c in C5 C4 C3; do python scripts/time_solve.py --config $c --log-errors --tag dense; MFADD_RES_ROWS=1 python scripts/time_solve.py --config $c --log-errors --tag rows; done
for kb in 140 90; do MFADD_RES_SMEM_KB=$kb python scripts/time_solve.py --config C5 --log-errors --tag "dense kb$kb"; done
