"""Debug helper: one small 2-D solve (kernel-by-kernel sync check via MFADD_SYNC_CHECK=1)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2210_06528_b200 as m
from paper_2210_06528_b200 import workloads as W
cfg = W.Config("t", (160, 150), (4, 4), 3, (10, 9), 3, "sinc_radial")
v = W.make_field_numpy(cfg)
dec = m.partition(cfg.grid, cfg.bounds, cfg.blocks, cfg.degree, cfg.nctrl, cfg.overlap)
s = m.Solver(dec, m.SolverConfig(max_outer_iterations=20, log_errors=False))
s.run(v.reshape(-1))
print("ok", s.result().constraint_iterations)
