#!/bin/bash
# Scan of tile / ring knobs on one config (graph-replay ms per solve):
#   bash scripts/knob_scan.sh C5
c=${1:-C5}
run() { env "$@" python scripts/time_solve.py --config $c --tag "$*"; }
run X=1
for v in 96 112 128 160 192 288; do run MFADD_AX0_COLS=$v; done
for v in 2 4; do run MFADD_FIT_S=$v; done
for v in 1 3 4; do run MFADD_LAST_SEGS=$v; done
for v in 2 3; do run MFADD_LAST_LSPLIT=$v; done
for v in 2 4; do run MFADD_DEC_S=$v; done
for v in 4 6 12 16; do run MFADD_DEC_CTAS=$v; done
for v in 2048 8192; do run MFADD_EPOCH_TILE=$v; done
for v in 0 1 2 5; do run MFADD_UNROLL_EPOCHS=$v; done
run MFADD_CHOL_INLINE=1
run MFADD_CHOL_HEAVY=1
run MFADD_NO_PDL=1
run X=1
