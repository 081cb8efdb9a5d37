"""Debug helper: run the configs that fail and report the failing stage."""
import sys
sys.path.insert(0, '.')
import paper_2210_06528_b200 as m
from paper_2210_06528_b200 import workloads as W
cfgs = [W.Config("odd2", (200, 199), (2, 3), 3, (20, 14), 3, "sinc_radial"),
        W.scaled(W.CONFIGS["C3"], (96, 100, 104), (12, 12, 13))]
for cfg in cfgs:
    v = W.make_field_numpy(cfg)
    dec = m.partition(cfg.grid, cfg.bounds, cfg.blocks, cfg.degree, cfg.nctrl, cfg.overlap)
    s = m.Solver(dec, m.SolverConfig(max_outer_iterations=20, log_errors=False))
    for it in range(3):
        try:
            s.run(v.reshape(-1))
            print(cfg.name, it, "ok", len(s.result().epochs))
        except Exception as e:
            print(cfg.name, it, "FAILED", e)
