set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "boundary or log_errors or shim or fit_singular" > gpurun_out/r2b_tests.log 2>&1; echo "tests rc=$?"
tail -30 gpurun_out/r2b_tests.log
for eg in 4 2; do MFADD_RES_EG=$eg timeout 300 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2b_C5_eg$eg.json 2> gpurun_out/r2b_C5_eg$eg.err; echo "C5 eg$eg rc=$?"; done
for eg in 4 2 1; do MFADD_RES_EG=$eg timeout 300 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2b_C4_eg$eg.json 2> gpurun_out/r2b_C4_eg$eg.err; echo "C4 eg$eg rc=$?"; done
