"""Debug helper: one loopback sharded solve with tracing."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2210_06528_b200 as m
from paper_2210_06528_b200 import workloads as W
cfg = W.scaled(W.CONFIGS["C2"], (400, 380), (20, 18))
v = W.make_field_numpy(cfg)
dec = m.partition(cfg.grid, cfg.bounds, cfg.blocks, cfg.degree, cfg.nctrl, cfg.overlap)
f = m.Field(list(cfg.grid), list(cfg.bounds), v)
sc = m.SolverConfig(max_outer_iterations=20, log_errors=False)
ref = m.solve(f, dec, sc)
print("single ok", ref.constraint_iterations, flush=True)
print("ranges", [m.shard_range(dec, r, 2) for r in range(2)], flush=True)
r = m.solve_loopback(f, dec, 2, sc)
print("loopback", r.constraint_iterations, np.abs(r.model.controls - ref.model.controls).max(), flush=True)
