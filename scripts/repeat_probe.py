"""Device time of a solve without the host round trip between solves: the
cached whole-solve graph enqueued K times back to back (mfadd_debug_solve_repeat)
against K solve() calls."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2210_06528_b200 as m  # noqa: E402
from paper_2210_06528_b200 import _lib as L  # noqa: E402
from paper_2210_06528_b200 import workloads as W  # noqa: E402

for name in sys.argv[1:] or ["C5"]:
    cfg = W.CONFIGS[name]
    field = W.make_field_torch(cfg)
    dec = m.partition(cfg.grid, cfg.bounds, cfg.blocks, cfg.degree, cfg.nctrl, cfg.overlap)
    st = torch.cuda.current_stream()
    ctx = m.Context(0, stream=st.cuda_stream)
    s = m.Solver(dec, m.SolverConfig(max_outer_iterations=cfg.max_iters, tolerance=cfg.tolerance,
                                     log_errors=False, store_error=True), ctx)
    for _ in range(3):
        s.run(field, on_device=True)
    lib = L.load()
    lib.mfadd_debug_solve_repeat.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
    K = 10
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(K):
        s.run(field, on_device=True)
    e1.record(st)
    torch.cuda.synchronize()
    a = e0.elapsed_time(e1) / K
    e0.record(st)
    lib.mfadd_debug_solve_repeat(s._h, C.c_void_p(field.data_ptr()), K)
    e1.record(st)
    torch.cuda.synchronize()
    b = e0.elapsed_time(e1) / K
    print(f"{name}: solve() x{K} {a:.4f} ms/solve, graph x{K} back to back {b:.4f} ms/solve", flush=True)
