"""Debug helper: repeated C2 solves through the whole-solve graph vs the oracle."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2210_06528_b200 as m
from paper_2210_06528_b200 import workloads as W
from oracle import orc
cfg = W.CONFIGS["C2"]
v = W.make_field_numpy(cfg)
dec = m.partition(cfg.grid, cfg.bounds, cfg.blocks, cfg.degree, cfg.nctrl, cfg.overlap)
s = m.Solver(dec, m.SolverConfig(max_outer_iterations=20, log_errors=False))
o = orc.solve(orc.Decomposition(cfg.grid, cfg.blocks, cfg.degree, cfg.nctrl, cfg.overlap), v, 20, 1e-10)
for it in range(4):
    try:
        s.run(v.reshape(-1))
    except Exception as e:
        print("run", it, "failed:", e)
        break
    g = s.result()
    d = max(np.abs(g.blocks[b].p - o.blocks_p[b]).max() for b in range(len(g.blocks)))
    print("run", it, "epochs", len(g.epochs), "iters", g.constraint_iterations, "maxdiff", d, "l2", g.global_l2)
