#!/bin/bash
# compute-sanitizer over a small solve of every kernel family (run under gpurun).
mkdir -p gpurun_out
for tool in racecheck memcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python scripts/solve_small.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/sanitize_$tool.log
done
