"""Debug helper: C2 fit (no epochs) with the TMA / generic passes vs the oracle."""
import os
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2210_06528_b200 as m
from paper_2210_06528_b200 import workloads as W
from oracle import orc
cfg = W.CONFIGS["C2"]
v = W.make_field_numpy(cfg)
dec = m.partition(cfg.grid, cfg.bounds, cfg.blocks, cfg.degree, cfg.nctrl, cfg.overlap)
s = m.Solver(dec, m.SolverConfig(max_outer_iterations=20, log_errors=False, enforce_continuity=False))
s.run(v.reshape(-1))
g = s.result()
o = orc.solve(orc.Decomposition(cfg.grid, cfg.blocks, cfg.degree, cfg.nctrl, cfg.overlap), v, 20, 1e-10,
              enforce_continuity=False)
for b in (0, 1, 5, 15):
    d = np.abs(g.blocks[b].p - o.blocks_p[b])
    bad = np.argwhere(d > 1e-9)
    print(os.environ.get("TAG"), "block", b, "maxdiff", d.max(), "bad", len(bad), bad[:3].tolist())
