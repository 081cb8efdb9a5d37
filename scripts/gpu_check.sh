#!/bin/bash
# One GPU batch of the round's checks (run under gpurun from the repo root):
# the GPU test suite, a timing of every BASELINE config through the graph path
# (both log_errors modes), and the default bench line.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/check_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/check_tests.log
for c in C5 C4 C3 C2 C1; do
  python scripts/time_solve.py --config $c --tag graph
  python scripts/time_solve.py --config $c --log-errors --tag graph
done
timeout 900 python bench.py > gpurun_out/check_bench.json 2> gpurun_out/check_bench.err; echo "bench rc=$?"
