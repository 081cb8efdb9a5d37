"""GPU path against the golden fixtures generated from the reference itself
(tests/golden/make_golden.py -> oracle/_ref).  Rows bit-exact, everything
else within 1e-10 relative (north_star tolerance)."""
import glob
import os

import numpy as np
import pytest

import paper_2210_06528_b200 as m
from tests.test_cpu_oracle import golden_values

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")
RTOL = 1e-10


def test_rows_golden(ctx):
    g = np.load(os.path.join(GOLD, "knots_collocation.npz"))
    for i in range(int(g["nkv"][0])):
        p, n, cl, cr = (int(x) for x in g[f"kv{i}_meta"])
        kv = m.make_knot_vector(p, n, 0.0, 1.0, bool(cl), bool(cr))
        bc = m.collocation_matrix(kv, g[f"kv{i}_params"], ctx=ctx)
        assert np.array_equal(bc.first_col, g[f"kv{i}_fc"])
        assert np.array_equal(bc.count, g[f"kv{i}_cnt"])
        assert np.array_equal(bc.values, g[f"kv{i}_vals"])


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "solve_*.npz"))),
                         ids=lambda p: os.path.basename(p)[6:-4])
def test_solve_golden_gpu(ctx, path):
    g = np.load(path)
    values = golden_values(g)
    p, ov, clamp, iters = int(g["degree"][0]), int(g["overlap"][0]), bool(g["clamp"][0]), int(g["max_iters"][0])
    grid = g["grid"].tolist()
    dec = m.partition(grid, [(0.0, 1.0)] * len(grid), g["blocks"].tolist(), p, g["nctrl"].tolist(), ov, clamp)
    assert np.array_equal(dec.block_dims_array(), g["blockdims"])
    bd = dec.block_dims_array()
    for b in (0, dec.nblocks - 1):  # block-problem rows, bit-exact
        for k in range(dec.rank):
            lo, hi = int(bd[b, k, 12]), int(bd[b, k, 13])
            u = np.array([j / (grid[k] - 1) for j in range(lo, hi)])
            bc = m.collocation_matrix(dec.kvs[k], u, int(bd[b, k, 8]), int(bd[b, k, 9]), ctx)
            assert np.array_equal(bc.first_col, g[f"rows_b{b}_d{k}_fc"])
            assert np.array_equal(bc.count, g[f"rows_b{b}_d{k}_cnt"])
            assert np.array_equal(bc.values, g[f"rows_b{b}_d{k}_vals"])
    s = m.Solver(dec, m.SolverConfig(max_outer_iterations=iters, tolerance=1e-10, log_errors=False), ctx)
    s.run(np.ascontiguousarray(values).reshape(-1))
    r = s.result()
    conv, ci, fdp, l2, linf = g["scalars"]
    assert r.converged == bool(conv) and r.constraint_iterations == int(ci)
    assert len(r.epochs) == len(g["epochs"])
    for e, ge in zip(r.epochs, g["epochs"]):
        for a, b in ((e.dp_max, ge[1]), (e.jump_ss, ge[2]), (e.jump_ms, ge[3])):
            assert abs(a - b) <= RTOL * max(1.0, abs(b))
    scale = max(1.0, float(np.abs(g["controls"]).max()))
    assert np.abs(r.model.controls - g["controls"]).max() <= RTOL * scale
    assert abs(r.global_l2 - l2) <= RTOL * max(1, l2) and abs(r.global_linf - linf) <= RTOL * max(1, linf)
    stride = int(g["global_error_stride"][0])
    assert np.abs(r.global_error.reshape(-1)[::stride] - g["global_error"]).max() <= RTOL * scale
    assert np.abs(r.blocks[0].p - g["block_p0"]).max() <= RTOL * scale
    assert np.abs(r.blocks[-1].p - g["block_plast"]).max() <= RTOL * scale
    fj = np.array([[j.block_a, j.block_b, j.linf_ss, j.linf_ms] for j in r.final_jumps]).reshape(-1, 4)
    assert fj.shape == g["final_jumps"].shape
    if fj.size:
        assert np.array_equal(fj[:, :2], g["final_jumps"][:, :2])
        assert np.abs(fj[:, 2:] - g["final_jumps"][:, 2:]).max() <= RTOL * scale
