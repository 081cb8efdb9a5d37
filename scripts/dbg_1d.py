"""Debug helper: 1-D single-device and loopback solves (C1)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2210_06528_b200 as m
from paper_2210_06528_b200 import workloads as W
cfg = W.CONFIGS["C1"]
v = W.make_field_numpy(cfg)
dec = m.partition(cfg.grid, cfg.bounds, cfg.blocks, cfg.degree, cfg.nctrl, cfg.overlap)
f = m.Field(list(cfg.grid), list(cfg.bounds), v)
sc = m.SolverConfig(max_outer_iterations=20, log_errors=False)
ref = m.solve(f, dec, sc)
print("single", ref.constraint_iterations, ref.global_l2, flush=True)
for n in (2, 4):
    r = m.solve_loopback(f, dec, n, sc)
    print("loopback", n, r.constraint_iterations, np.abs(r.model.controls - ref.model.controls).max(), r.global_l2,
          flush=True)
