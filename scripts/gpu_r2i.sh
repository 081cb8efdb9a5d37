mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak scripts/probes/fp64_peak.cu && /tmp/fp64_peak > gpurun_out/fp64_peak.json; cat gpurun_out/fp64_peak.json
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2i_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2i_tests.log
timeout 900 python bench.py > gpurun_out/r2i_bench.json 2> gpurun_out/r2i_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/r2i_ref.json 2> gpurun_out/r2i_ref.err; echo "ref rc=$?"
timeout 600 compute-sanitizer --tool racecheck --racecheck-report hazard python scripts/solve_small.py > gpurun_out/r2i_racecheck.log 2>&1; echo "racecheck rc=$?"; tail -5 gpurun_out/r2i_racecheck.log
