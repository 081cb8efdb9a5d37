# decode geometry sweep (bench.py C5): MFADD_DEC_MINB launch-bounds min blocks, MFADD_DEC_CTAS row ranges per SM
for cfg in "$@"; do set -- $cfg; MFADD_DEC_MINB=$1 MFADD_DEC_CTAS=$2 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/dec_$1_$2.log 2>&1; done
