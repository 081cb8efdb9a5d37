"""Per-kernel CUDA-event times of one BASELINE config (direct launches, an
event pair around every launch; averages over --steps solves).

    python scripts/kernel_times.py --config C5 [--log-errors]
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
dec = m.partition(cfg.grid, cfg.bounds, cfg.blocks, cfg.degree, cfg.nctrl, cfg.overlap)
st = torch.cuda.current_stream()
ctx = m.Context(0, stream=st.cuda_stream)
s = m.Solver(dec, m.SolverConfig(max_outer_iterations=cfg.max_iters, tolerance=cfg.tolerance,
                                 log_errors=args.log_errors, store_error=True), ctx)
for _ in range(3):
    s.run(field, on_device=True)
s.set_profiling(True)
for _ in range(args.steps):
    s.run(field, on_device=True)
torch.cuda.synchronize()
acc = {}
for name, ms in s.kernel_times():
    acc.setdefault(name, []).append(ms)
print(args.tag, cfg.name, " ".join(f"{k}={1e3 * sum(v) / args.steps:.1f}us" for k, v in acc.items()), flush=True)
