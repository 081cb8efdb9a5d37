import sys; sys.path.insert(0,'.')
import numpy as np
import paper_2210_06528_b200 as m
from paper_2210_06528_b200 import workloads as W
cfg = W.scaled(W.CONFIGS["C3"], (40, 44, 48), (8, 9, 10))
cfg = W.Config("t", cfg.grid, (2,2,2), 3, (8,9,10), 3, "sinc_radial")
v = W.make_field_numpy(cfg)
dec = m.partition(cfg.grid, cfg.bounds, cfg.blocks, cfg.degree, cfg.nctrl, cfg.overlap)
s = m.Solver(dec, m.SolverConfig(max_outer_iterations=20, log_errors=False))
s.run(v.reshape(-1)); print("ok", s.result().constraint_iterations)
