"""Time K whole-solve graph replays of one BASELINE config (A/B of knobs).

    python scripts/time_solve.py --config C5 [--log-errors] [--steps 10]
prints one line: config, log_errors, ms per solve (CUDA events), epochs.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--log-errors", action="store_true")
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--tag", default="")
args = ap.parse_args()

import torch  # noqa: E402

import paper_2210_06528_b200 as m  # noqa: E402
from paper_2210_06528_b200 import workloads as W  # noqa: E402

cfg = W.CONFIGS[args.config]
field = W.make_field_torch(cfg)
torch.cuda.synchronize()
dec = m.partition(cfg.grid, cfg.bounds, cfg.blocks, cfg.degree, cfg.nctrl, cfg.overlap)
st = torch.cuda.current_stream()
ctx = m.Context(0, stream=st.cuda_stream)
s = m.Solver(dec, m.SolverConfig(max_outer_iterations=cfg.max_iters, tolerance=cfg.tolerance,
                                 log_errors=args.log_errors, store_error=True), ctx)
for _ in range(3):
    s.run(field, on_device=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(args.steps):
    s.run(field, on_device=True)
e1.record(st)
torch.cuda.synchronize()
r = s.result(want_blocks=False, want_error=False)
print(f"{args.tag} {cfg.name} log_errors={int(args.log_errors)} ms={e0.elapsed_time(e1) / args.steps:.4f} "
      f"epochs={len(r.epochs)} l2={r.global_l2:.6e}", flush=True)
