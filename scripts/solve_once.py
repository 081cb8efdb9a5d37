"""Run N solves of one BASELINE config on cuda:0 (profiling target for ncu).

    python scripts/solve_once.py --config C4 [--log-errors] [--steps 1] [--warmup 0]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--log-errors", action="store_true")
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--warmup", type=int, default=0)
args = ap.parse_args()

import torch  # noqa: E402

import paper_2210_06528_b200 as m  # noqa: E402
from paper_2210_06528_b200 import workloads as W  # noqa: E402

cfg = W.CONFIGS[args.config]
field = W.make_field_torch(cfg)
torch.cuda.synchronize()
dec = m.partition(cfg.grid, cfg.bounds, cfg.blocks, cfg.degree, cfg.nctrl, cfg.overlap)
ctx = m.Context(0, stream=torch.cuda.current_stream().cuda_stream)
solver = m.Solver(dec, m.SolverConfig(max_outer_iterations=cfg.max_iters, tolerance=cfg.tolerance,
                                      log_errors=args.log_errors, store_error=True), ctx)
for _ in range(args.warmup + args.steps):
    solver.run(field, on_device=True)
torch.cuda.synchronize()
r = solver.result(want_blocks=False, want_error=False)
print(f"{cfg.name} iters={r.constraint_iterations} epochs={len(r.epochs)} l2={r.global_l2:.6e} linf={r.global_linf:.6e}")
