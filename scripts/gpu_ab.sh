#!/bin/bash
# A/B of an environment knob on the graph-replay timings (run under gpurun):
#   bash scripts/gpu_ab.sh MFADD_NO_TWIST C5 C2
knob=$1; shift
for c in "$@"; do
  python scripts/time_solve.py --config $c --tag "default"
  env $knob=1 python scripts/time_solve.py --config $c --tag "$knob=1"
done
