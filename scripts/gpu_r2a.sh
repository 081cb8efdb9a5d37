set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2a_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r2a_tests.log
for c in C5 C3 C4 C2 C1; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2a_bench_$c.json 2> gpurun_out/r2a_bench_$c.err; echo "$c rc=$?"; done
