#!/bin/bash
# Round evidence batch (run under gpurun): gpu_check.sh, then the launch list
# and ncu --set full captures of C5 (both log_errors modes), C4 and C3, and
# the sharded / legacy-residual paths under their knobs.
bash scripts/gpu_check.sh
MFADD_HOST_LOOP=1 MFADD_RES_LEGACY=1 timeout 600 python -m pytest tests/test_gpu_parity.py -k "log_errors" -m gpu -q 2>&1 | tail -2
bash scripts/profile_round.sh || echo "profile_round failed"
for c in C4 C3; do bash scripts/profile_config.sh $c || echo "profile $c failed"; done
bash scripts/profile_config.sh C5 --log-errors || echo "profile C5 le failed"
bash scripts/profile_config.sh C4 --log-errors || echo "profile C4 le failed"
