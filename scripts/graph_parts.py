"""Whole-solve graph time of C5 with and without the continuity epochs
(enforce_continuity), and without the error field: what the epoch loop and
the error write cost inside the graph (kernel-level profiling cannot see
into graphs with conditional nodes)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2210_06528_b200 as m  # noqa: E402
from paper_2210_06528_b200 import workloads as W  # noqa: E402

cfg = W.CONFIGS["C5"]
field = W.make_field_torch(cfg).contiguous()
dec = m.partition(cfg.grid, cfg.bounds, cfg.blocks, cfg.degree, cfg.nctrl, cfg.overlap)


def t(enforce, store_error, reps=10):
    s = m.Solver(dec, m.SolverConfig(max_outer_iterations=20, tolerance=1e-10, log_errors=False,
                                      enforce_continuity=enforce, store_error=store_error))
    for _ in range(3):
        s.run(field, on_device=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        s.run(field, on_device=True)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for enforce in (True, False):
    for err in (True, False):
        print(f"enforce={enforce} store_error={err}: {t(enforce, err):.4f} ms")
