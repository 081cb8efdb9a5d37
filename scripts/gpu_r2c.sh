set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "boundary or log_errors or shim or fit_singular" > gpurun_out/r2c_tests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/r2c_tests.log
timeout 300 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline --no-other > gpurun_out/r2c_C5.json 2> gpurun_out/r2c_C5.err; echo "C5 rc=$?"
timeout 300 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-other > gpurun_out/r2c_C4.json 2> gpurun_out/r2c_C4.err; echo "C4 rc=$?"
timeout 300 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-other > gpurun_out/r2c_C3.json 2> gpurun_out/r2c_C3.err; echo "C3 rc=$?"
NCU_K="k_residual|k_epoch_regions|k_decode" NCU_COUNT=8 bash scripts/profile_config.sh C5 --log-errors
NCU_K="k_residual|k_decode|k_fit|k_last|k_axis0" NCU_COUNT=10 bash scripts/profile_config.sh C4 --log-errors
