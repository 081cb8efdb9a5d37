"""A small solve of every kernel family (2-D and 3-D, log_errors on) for
compute-sanitizer runs (racecheck / memcheck)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2210_06528_b200 as m  # noqa: E402
from paper_2210_06528_b200 import workloads as W  # noqa: E402

for cfg in (W.scaled(W.CONFIGS["C5"], (384, 352), (24, 22)),
            W.Config("C4t", (96, 90, 88), (2, 2, 2), 4, (13, 13, 13), 4, "combustion")):
    values = W.make_field_numpy(cfg)
    dec = m.partition(cfg.grid, cfg.bounds, cfg.blocks, cfg.degree, cfg.nctrl, cfg.overlap)
    s = m.Solver(dec, m.SolverConfig(max_outer_iterations=20, log_errors=True, store_error=True))
    for _ in range(2):
        s.run(values.reshape(-1))
    r = s.result(want_blocks=False, want_error=False)
    print(cfg.name, r.constraint_iterations, len(r.epochs), r.global_l2, np.array(r.epochs[-1].block_errors).max())
    s.close()
