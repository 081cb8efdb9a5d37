"""C5 with log_errors=true: whole-solve time, and (under ncu, MFADD_HOST_LOOP=1)
one solve's direct launches, to see what the per-epoch block residuals cost."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2210_06528_b200 as m  # noqa: E402
from paper_2210_06528_b200 import workloads as W  # noqa: E402

cfg = W.CONFIGS["C5"]
field = W.make_field_torch(cfg).contiguous()
dec = m.partition(cfg.grid, cfg.bounds, cfg.blocks, cfg.degree, cfg.nctrl, cfg.overlap)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
for le in (False, True):
    s = m.Solver(dec, m.SolverConfig(max_outer_iterations=20, tolerance=1e-10, log_errors=le))
    for _ in range(min(reps, 3)):
        s.run(field, on_device=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        s.run(field, on_device=True)
    e1.record()
    torch.cuda.synchronize()
    print(f"log_errors={le}: {e0.elapsed_time(e1) / reps:.4f} ms", flush=True)
    s.close()
