mkdir -p gpurun_out
python scripts/time_solve.py --config C5 --tag base
for kb in 110 80 64; do for eg in 4 2; do MFADD_RES_SMEM_KB=$kb MFADD_RES_EG=$eg python scripts/time_solve.py --config C5 --log-errors --tag "kb$kb eg$eg"; done; done
python scripts/time_solve.py --config C4 --tag base
for kb in 110 64; do for eg in 4 2; do MFADD_RES_SMEM_KB=$kb MFADD_RES_EG=$eg python scripts/time_solve.py --config C4 --log-errors --steps 3 --tag "kb$kb eg$eg"; done; done
timeout 600 python -m pytest tests -m gpu -x -q -k "log_errors or sharded or loopback" 2>&1 | tail -3
