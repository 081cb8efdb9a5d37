set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "log_errors" > gpurun_out/r2d_tests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/r2d_tests.log
for c in C5 C4 C3; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-other > gpurun_out/r2d_$c.json 2> gpurun_out/r2d_$c.err; echo "$c rc=$?"; done
NCU_K="k_residual" NCU_COUNT=1 bash scripts/profile_config.sh C5 --log-errors
NCU_K="k_residual" NCU_COUNT=1 bash scripts/profile_config.sh C4 --log-errors
timeout 1200 python -m pytest tests -m gpu -x -q -k "fullsize" > gpurun_out/r2d_full.log 2>&1; echo "full rc=$?"
tail -30 gpurun_out/r2d_full.log
