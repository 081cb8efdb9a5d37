"""Full-size BASELINE configs against the reference itself (oracle/_ref, the
unmodified sources compiled by oracle/Makefile), on the identical field
buffer (the device generator's output copied to the host):

  C3  256^3 radial sinc, 4^3 blocks, p=3, 32^3 controls/block, overlap 3
  C4  704x540x550 combustion-shaped field, 8^3 blocks, p=4, 24^3 controls/block, overlap 4
  C5  8192^2 radial sinc, 16^2 blocks, p=5, 128^2 controls/block, overlap 5

Checked: every block's collocation rows bit-exact
(spans via first_col, count, basis values) on the solver's own axis problems;
the global lattice max|dP| <= 1e-10 * max(1, ||P_ref||_inf); L2 / L-inf within
1e-10 relative; converged, constraint_iterations and the epoch count equal;
per-epoch dp / SS / MS jumps within 1e-10; the final per-pair jumps; the
pointwise error field within 1e-10; and with log_errors the per-epoch block
residuals within 1e-10 (solver.cpp:332-440, decode.cpp:83-97, lsq.cpp:66-85).

The reference solve of C4 takes tens of seconds on the host's cores.
"""
import os

import numpy as np
import pytest

import paper_2210_06528_b200 as m
from oracle import ref
from paper_2210_06528_b200 import workloads as W

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

RTOL = 1e-10
needs_ref = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")


def _close(a, b):
    scale = max(1.0, float(np.abs(b).max()))
    return float(np.abs(a - b).max()) <= RTOL * scale, float(np.abs(a - b).max()) / scale


def _rows_bit_exact(cfg, dec, ctx):
    """K1 on exactly the solver's axis problems (one per (dim, block coordinate))
    against the reference collocation_matrix (collocation.cpp:83-111)."""
    bd = dec.block_dims_array()
    coords = np.array([b.coords for b in dec.blocks])
    for k in range(dec.rank):
        kv = dec.kvs[k]
        M = cfg.grid[k]
        for c in range(cfg.blocks[k]):
            b = int(np.nonzero(coords[:, k] == c)[0][0])
            lo, hi = int(bd[b, k, 8]), int(bd[b, k, 9])
            i0, i1 = int(bd[b, k, 12]), int(bd[b, k, 13])
            u = np.arange(i0, i1, dtype=np.float64) / float(M - 1)
            g = m.collocation_matrix(kv, u, lo, hi, ctx)
            ofc, ocnt, ovals = ref.collocation(kv.knots, cfg.degree, u, lo, hi)
            assert np.array_equal(g.first_col, ofc), (k, c)
            assert np.array_equal(g.count, ocnt), (k, c)
            assert np.array_equal(g.values, ovals), (k, c)


@needs_ref
@pytest.mark.parametrize("name", ["C3", "C4", "C5"])
def test_fullsize_vs_reference(ctx, name):
    import torch
    cfg = W.CONFIGS[name]
    field = W.make_field_torch(cfg)
    host = field.cpu().numpy()
    dec = m.partition(cfg.grid, cfg.bounds, cfg.blocks, cfg.degree, cfg.nctrl, cfg.overlap)
    _rows_bit_exact(cfg, dec, ctx)
    s = m.Solver(dec, m.SolverConfig(max_outer_iterations=cfg.max_iters, tolerance=cfg.tolerance,
                                     log_errors=True, store_error=True), ctx)
    s.run(field, on_device=True)
    s.run(field, on_device=True)  # the whole-solve graph (capture) ...
    s.run(field, on_device=True)  # ... and its replay
    g = s.result(want_blocks=False, want_error=True)
    s.close()
    del field
    torch.cuda.empty_cache()
    rd = ref.RefDecomposition(cfg.grid, cfg.blocks, cfg.degree, cfg.nctrl, cfg.overlap,
                              bounds=[list(b) for b in cfg.bounds])
    r = ref.solve(rd, host, cfg.max_iters, cfg.tolerance, workers=os.cpu_count() or 1, log_errors=True,
                  want_blocks=False)
    assert g.converged == r.converged
    assert g.constraint_iterations == r.constraint_iterations
    assert len(g.epochs) == len(r.epochs)
    for ge, oe in zip(g.epochs, r.epochs):
        assert ge.iteration == int(oe[0])
        for gv, ov in ((ge.dp_max, oe[1]), (ge.jump_ss, oe[2]), (ge.jump_ms, oe[3])):
            assert abs(gv - ov) <= RTOL * max(1.0, abs(ov)), (name, ge, oe)
    ok, dp = _close(g.model.controls, r.controls)
    assert ok, (name, dp)
    assert abs(g.global_l2 - r.global_l2) <= RTOL * max(1.0, r.global_l2)
    assert abs(g.global_linf - r.global_linf) <= RTOL * max(1.0, r.global_linf)
    ok, de = _close(g.global_error, r.global_error)
    assert ok, (name, de)
    assert len(g.final_jumps) == len(r.final_jumps)
    for gj, oj in zip(g.final_jumps, r.final_jumps):
        assert (gj.block_a, gj.block_b) == (int(oj[0]), int(oj[1]))
        assert abs(gj.linf_ss - oj[2]) <= RTOL * max(1.0, oj[2])
        assert abs(gj.linf_ms - oj[3]) <= RTOL * max(1.0, oj[3])
    assert len(r.block_errors) == len(g.epochs)
    for ge, ob in zip(g.epochs, r.block_errors):
        got = np.array(ge.block_errors)
        want = np.asarray(ob).reshape(got.shape)
        assert np.all(np.abs(got - want) <= RTOL * np.maximum(1.0, np.abs(want))), (name, ge.iteration)
