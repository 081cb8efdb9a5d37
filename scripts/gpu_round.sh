#!/bin/bash
# Round evidence batch (run under gpurun): gpu_check.sh, then the launch list
# and ncu --set full captures of C5 (both log_errors modes), C4 and C3.
bash scripts/gpu_check.sh
bash scripts/profile_round.sh || echo "profile_round failed"
for c in C4 C3; do bash scripts/profile_config.sh $c || echo "profile $c failed"; done
bash scripts/profile_config.sh C5 --log-errors || echo "profile C5 le failed"
bash scripts/profile_config.sh C4 --log-errors || echo "profile C4 le failed"
