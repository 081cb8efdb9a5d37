# last-axis contraction segment-count sweep (bench.py C5)
for k in "$@"; do MFADD_LAST_SEGS=$k timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/seg_$k.log 2>&1; done
