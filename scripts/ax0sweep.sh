# axis-0 tile geometry sweep (bench.py C5): MFADD_AX0_COLS columns per CTA, MFADD_FIT_S TMA stages
for cfg in "$@"; do set -- $cfg; MFADD_AX0_COLS=$1 MFADD_FIT_S=$2 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ax_$1_$2.log 2>&1; done
