"""GPU parity: the CUDA path (through the C ABI) against the C oracle
restatement (oracle/liboracle.so), on identical seeded inputs.

Tolerances (north_star): spans / first_col / count bit-exact; basis values and
Gram entries bit-exact (explicit RN arithmetic); control points and decoded
values within 1e-10 relative: max|dP| <= 1e-10 * max(1, ||P_ref||_inf).
"""
import math

import numpy as np
import pytest

import paper_2210_06528_b200 as m
from oracle import orc
from paper_2210_06528_b200 import workloads as W

pytestmark = pytest.mark.gpu

RTOL = 1e-10


def close(a, b, rtol=RTOL):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    scale = max(1.0, float(np.abs(b).max()) if b.size else 1.0)
    return float(np.abs(a - b).max()) <= rtol * scale if b.size else True


def run_both(cfg, values, max_iters=None, tol=None, enforce=True):
    dec = m.partition(cfg.grid, cfg.bounds, cfg.blocks, cfg.degree, cfg.nctrl, cfg.overlap)
    sc = m.SolverConfig(max_outer_iterations=max_iters or cfg.max_iters, tolerance=tol or cfg.tolerance,
                        log_errors=False, enforce_continuity=enforce, store_error=True)
    s = m.Solver(dec, sc)
    s.run(values.reshape(-1))
    g = s.result()
    od = orc.Decomposition(cfg.grid, cfg.blocks, cfg.degree, cfg.nctrl, cfg.overlap)
    o = orc.solve(od, values, max_outer_iterations=sc.max_outer_iterations, tolerance=sc.tolerance,
                  enforce_continuity=enforce)
    return g, o, s


def assert_solve_parity(g, o):
    assert g.converged == o.converged
    assert g.constraint_iterations == o.constraint_iterations
    assert len(g.epochs) == len(o.epochs)
    for ge, oe in zip(g.epochs, o.epochs):
        assert ge.iteration == int(oe[0])
        for gv, ov in ((ge.dp_max, oe[1]), (ge.jump_ss, oe[2]), (ge.jump_ms, oe[3])):
            assert abs(gv - ov) <= RTOL * max(1.0, abs(ov)), (ge, oe)
    assert close(g.model.controls, o.controls)
    for gb, ob in zip(g.blocks, o.blocks_p):
        assert gb.p.shape == ob.shape
        assert close(gb.p, ob)
    assert abs(g.global_l2 - o.global_l2) <= RTOL * max(1.0, o.global_l2)
    assert abs(g.global_linf - o.global_linf) <= RTOL * max(1.0, o.global_linf)
    assert close(g.global_error, o.global_error)
    assert len(g.final_jumps) == len(o.final_jumps)
    for gj, oj in zip(g.final_jumps, o.final_jumps):
        assert (gj.block_a, gj.block_b) == (int(oj[0]), int(oj[1]))
        assert abs(gj.linf_ss - oj[2]) <= RTOL * max(1.0, oj[2])
        assert abs(gj.linf_ms - oj[3]) <= RTOL * max(1.0, oj[3])


# ------------------------------------------------------------------ K1 rows


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 7, 9])
def test_collocation_rows_bit_exact(ctx, p):
    rng = np.random.default_rng(20240811 + p)
    for clamp in [(True, True), (True, False), (False, True), (False, False)]:
        n = p + 1 + int(rng.integers(0, 40))
        kv = m.make_knot_vector(p, n, 0.0, 1.0, *clamp)
        okn = orc.make_knot_vector(p, n, 0.0, 1.0, *clamp)
        assert np.array_equal(kv.knots, okn)
        params = np.sort(rng.uniform(kv.domain_min(), kv.domain_max(), 300))
        params[0], params[-1] = kv.domain_min(), kv.domain_max()
        lo = int(rng.integers(0, max(1, n // 3)))
        hi = int(n - rng.integers(0, max(1, n // 3)))
        # keep only params with an active basis in the window (else the reference throws)
        fc, cnt, vals = orc.collocation(kv.knots, p, params)
        spans = fc + p
        keep = (np.minimum(spans + 1, hi) - np.maximum(spans - p, lo)) > 0
        params = params[keep]
        if len(params) == 0:
            continue
        g = m.collocation_matrix(kv, params, lo, hi, ctx)
        ofc, ocnt, ovals = orc.collocation(kv.knots, p, params, lo, hi)
        assert np.array_equal(g.first_col, ofc)
        assert np.array_equal(g.count, ocnt)
        assert np.array_equal(g.values, ovals)  # bit-exact (explicit RN Cox-de Boor)


@pytest.mark.parametrize("p", [2, 3, 5])
def test_collocation_nonuniform_knots_bit_exact(ctx, p):
    """Spans on strongly non-uniform knots with repeated interior knots: the
    device's uniform-spacing guess must hand over to the binary search and
    land on the reference's span (knots.cpp:83-106) every time."""
    rng = np.random.default_rng(7 + p)
    for trial in range(4):
        inner = np.sort(rng.uniform(0.0, 1.0, 30) ** (1 + 3 * trial))  # clustered toward 0
        inner = np.concatenate([inner, inner[5:8]])                     # repeated knots
        inner.sort()
        kn = np.concatenate([[0.0] * (p + 1), inner, [1.0] * (p + 1)])
        kv = m.KnotVector(p, kn)
        params = np.sort(np.concatenate([rng.uniform(0.0, 1.0, 400), inner, [0.0, 1.0]]))
        g = m.collocation_matrix(kv, params, ctx=ctx)
        ofc, ocnt, ovals = orc.collocation(kn, p, params)
        assert np.array_equal(g.first_col, ofc)
        assert np.array_equal(g.count, ocnt)
        assert np.array_equal(g.values, ovals)


def test_collocation_known_answers(ctx):
    # test_collocation.cpp:13-21
    kv = m.make_knot_vector(2, 3, 0.0, 1.0)
    d = m.collocation_matrix(kv, [0.0, 0.5, 1.0], ctx=ctx).dense()
    assert np.allclose(d.reshape(-1), [1, 0, 0, 0.25, 0.5, 0.25, 0, 0, 1], rtol=0, atol=1e-14)
    # knots.cpp find_span conventions (test_knots.cpp:37-46)
    kv = m.KnotVector(2, np.array([0, 0, 0, 0.5, 1, 1, 1.0]))
    assert m.find_span(kv, 0.25, ctx) == 2
    assert m.find_span(kv, 1.0, ctx) == 3
    assert m.find_span(kv, 0.5, ctx) == 3
    with pytest.raises(m.OutOfRange):
        m.find_span(kv, 1.5, ctx)
    with pytest.raises(m.OutOfRange):
        m.find_span(kv, -0.1, ctx)
    # rejects bad parameter lists (test_collocation.cpp:45-49)
    kv = m.make_knot_vector(2, 5)
    with pytest.raises(m.InvalidArgument):
        m.collocation_matrix(kv, [0.5, 0.25], ctx=ctx)
    with pytest.raises(m.OutOfRange):
        m.collocation_matrix(kv, [0.0, 1.25], ctx=ctx)
    # window clipping (test_collocation.cpp:51-65)
    kv = m.make_knot_vector(3, 12)
    params = [j / 30.0 * 0.55 for j in range(31)]
    g = m.collocation_matrix(kv, params, 0, 7, ctx)
    assert g.cols == 7
    trunc = [j for j in range(g.rows) if g.count[j] < 4]
    assert trunc and all(g.row_sum(j) < 1 - 1e-12 for j in trunc)


# ------------------------------------------------------------------ K2+K3 fit


def _uniform(mm):
    return np.array([j / (mm - 1) for j in range(mm)])


@pytest.mark.parametrize("d", [1, 2, 3])
def test_fit_unconstrained_vs_oracle(ctx, d):
    rng = np.random.default_rng(5150 + d)
    for p in (2, 3, 4, 5):
        kvs, params, wins = [], [], []
        for k in range(d):
            n = p + 1 + int(rng.integers(4, 14))
            kv = m.make_knot_vector(p, n)
            mm = n + int(rng.integers(0, 3 * n)) + 3
            kvs.append(kv)
            params.append(_uniform(mm))
            wins.append((0, n))
        q = rng.uniform(-1, 1, tuple(len(pp) for pp in params))
        g = m.fit_unconstrained(m.LocalProblem(kvs, params, wins, q), ctx)
        o = orc.fit_unconstrained([k.knots for k in kvs], p, params, wins, q)
        assert close(g, o), (d, p, np.abs(g - o).max())


def test_fit_windowed_truncated(ctx):
    # clipped (truncated) windows as in the solver's block problems
    p = 3
    kv = m.make_knot_vector(p, 40)
    params = [np.arange(300, 700) / 999.0, np.arange(100, 420) / 999.0]
    wins = [(12, 27), (4, 17)]
    q = np.random.default_rng(7).standard_normal((400, 320))
    g = m.fit_unconstrained(m.LocalProblem([kv, kv], params, wins, q), ctx)
    o = orc.fit_unconstrained([kv.knots, kv.knots], p, params, wins, q)
    assert close(g, o)


def test_fit_bitwise_deterministic(ctx):
    # test_lsq.cpp:182-189
    kv = m.make_knot_vector(3, 12)
    prm = _uniform(64)
    q = np.exp(np.sin(9.0 * prm))
    a = m.fit_unconstrained(m.LocalProblem([kv], [prm], [(0, 12)], q), ctx)
    b = m.fit_unconstrained(m.LocalProblem([kv], [prm], [(0, 12)], q), ctx)
    assert np.array_equal(a, b)


def test_fit_singular_and_underdetermined(ctx):
    # test_lsq.cpp:191-215
    kv = m.make_knot_vector(2, 8)
    params = [0.3 * j / 10.0 for j in range(11)]
    with pytest.raises(m.SingularFitError) as ei:
        m.fit_unconstrained(m.LocalProblem([kv], [np.array(params)], [(0, 8)], np.ones(11)), ctx)
    # u <= 0.27 lies in knot spans [0, 1/6) and [1/6, 1/3): columns 0..3 supported,
    # the first uncovered one (uncovered_column, lsq.cpp:25-35) is 4
    assert ei.value.dim == 0 and ei.value.span == 4
    with pytest.raises(m.InvalidArgument):
        m.fit_unconstrained(m.LocalProblem([kv], [_uniform(5)], [(0, 8)], np.zeros(5)), ctx)


def test_polynomial_reproduction(ctx):
    # test_lsq.cpp:80-101
    for p in (2, 3):
        kv = m.make_knot_vector(p, 8)
        u0, u1 = _uniform(17), _uniform(15)

        def poly(x):
            return 0.7 + sum((0.3 + 0.1 * k) * x ** k for k in range(1, p + 1))
        q = np.outer(poly(u0), poly(u1))
        P = m.fit_unconstrained(m.LocalProblem([kv, kv], [u0, u1], [(0, 8), (0, 8)], q), ctx)
        dec = m.decode(P, [kv, kv], [u0, u1], ctx=ctx)
        assert np.abs(dec - q).max() < 1e-9


# ------------------------------------------------------------------ K7 decode


@pytest.mark.parametrize("d", [1, 2, 3])
def test_decode_vs_oracle(ctx, d):
    rng = np.random.default_rng(99 + d)
    for p in (1, 3, 5):
        kvs, params, ext = [], [], []
        for k in range(d):
            n = p + 1 + int(rng.integers(2, 12))
            kv = m.make_knot_vector(p, n)
            kvs.append(kv)
            params.append(np.sort(rng.uniform(0, 1, int(rng.integers(5, 40)))))
            ext.append(n)
        P = rng.standard_normal(tuple(ext))
        g = m.decode(P, kvs, params, ctx=ctx)
        o = orc.decode(P, [k.knots for k in kvs], p, params)
        assert np.abs(g - o).max() <= 1e-12 * max(1.0, np.abs(o).max())


def test_decode_windowed(ctx):
    p = 3
    kv = m.make_knot_vector(p, 30)
    params = [np.linspace(0.35, 0.6, 41)]
    P = np.random.default_rng(3).standard_normal(14)
    g = m.decode(P, [kv], params, col_offset=[9], ctx=ctx)
    o = orc.decode(P, [kv.knots], p, params, col_offset=[9])
    assert np.abs(g - o).max() <= 1e-12


# ------------------------------------------------------------------ solve


# Scaled families keep every block at least 2(floor(p/2)+overlap) spans wide,
# so each control has <= 2 holders per axis (the reference throws otherwise;
# see test_three_holder_fault), and keep the parent's inputs-per-control
# ratio (C3 2.0, C4 ~3.7, C5 4.0) so the local problems stay as well
# conditioned as at full size.
SMALL = {
    "C1": W.CONFIGS["C1"],  # full size: 10,000 points
    "C2": W.CONFIGS["C2"],  # full size: 1024^2
    "C3s": W.scaled(W.CONFIGS["C3"], (96, 100, 104), (12, 12, 13)),
    "C4s": W.Config("C4s", (190, 186, 182), (4, 4, 4), 4, (13, 13, 13), 4, "combustion"),
    "C5s": W.scaled(W.CONFIGS["C5"], (1536, 1408), (24, 22)),
}


@pytest.mark.parametrize("name", list(SMALL))
def test_solve_parity(ctx, name):
    cfg = SMALL[name]
    values = W.make_field_numpy(cfg)
    g, o, _ = run_both(cfg, values)
    assert_solve_parity(g, o)


def test_three_holder_fault(ctx):
    """Blocks narrower than 2(floor(p/2)+overlap) spans: a control has a holder
    two coordinates away, which never hears from it; the reference throws
    runtime_error from enforce_constraints (solver.cpp:134-141)."""
    cfg = W.scaled(W.CONFIGS["C3"], (64, 72, 80), (8, 9, 10))
    values = W.make_field_numpy(cfg)
    od = orc.Decomposition(cfg.grid, cfg.blocks, cfg.degree, cfg.nctrl, cfg.overlap)
    with pytest.raises(orc.OracleError) as oe:
        orc.solve(od, values, 20, 1e-10)
    dec = m.partition(cfg.grid, cfg.bounds, cfg.blocks, cfg.degree, cfg.nctrl, cfg.overlap)
    with pytest.raises(m.RuntimeFault) as ge:
        m.Solver(dec, m.SolverConfig(max_outer_iterations=20, log_errors=False)).run(values.reshape(-1))
    assert str(ge.value) == str(oe.value).split("] ", 1)[1]
    # without continuity enforcement the reference completes: decoupled fits,
    # epoch-0 jumps over neighbour pairs only, final per-pair jumps
    g, o, _ = run_both(cfg, values, enforce=False)
    assert_solve_parity(g, o)


def test_solve_known_answers(ctx):
    # test_solver.cpp:169-205 on the reference's own generators
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    f = ref.gen_field("sinc1d-asym", [2000])
    dec = m.partition([2000], [(-4, 4)], [2], 3, [30], 3)
    r = m.solve(m.Field([2000], [(-4, 4)], f), dec, m.SolverConfig(workers=2, log_errors=False))
    assert r.converged and r.constraint_iterations == 1 and len(r.epochs) == 3
    assert r.epochs[0].jump_ss > 1e-12 and r.epochs[1].dp_max > 0.0
    assert r.epochs[1].jump_ss < 1e-12 and r.epochs[2].dp_max < 1e-10
    assert all(j.linf_ss < 1e-12 and j.linf_ms == 0.0 for j in r.final_jumps)
    f = ref.gen_field("sinc2d", [64, 64])
    dec = m.partition([64, 64], [(-4, 4)] * 2, [2, 2], 3, [12, 12], 0)
    r = m.solve(m.Field([64, 64], [(-4, 4)] * 2, f), dec, m.SolverConfig(log_errors=False))
    assert r.converged and r.constraint_iterations == 2 and len(r.epochs) == 4
    assert r.epochs[1].jump_ss < 1e-12 and r.epochs[1].jump_ms > 1e-12
    assert r.epochs[2].jump_ss < 1e-12 and r.epochs[2].jump_ms < 1e-12
    assert r.epochs[2].dp_max > 0.0 and r.epochs[3].dp_max < 1e-10
    # non-convergence reporting (test_solver.cpp:301-310)
    r = m.solve(m.Field([64, 64], [(-4, 4)] * 2, f), dec, m.SolverConfig(max_outer_iterations=1, log_errors=False))
    assert not r.converged and r.constraint_iterations == 1 and r.final_dp >= 1e-10
    # single block: zero exchange epochs (test_solver.cpp:207-214)
    f = ref.gen_field("sinc1d-sym", [400])
    dec = m.partition([400], [(-4, 4)], [1], 3, [40], 0)
    r = m.solve(m.Field([400], [(-4, 4)], f), dec, m.SolverConfig(log_errors=False))
    assert r.converged and r.constraint_iterations == 0 and len(r.epochs) == 1


def test_solve_vs_reference_library(ctx):
    """Direct pin against the reference implementation itself (oracle/_ref)."""
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    for gen, npts, blocks, p, nc, ov in [("sinc2d", [72, 72], [3, 3], 3, [8, 8], 1),
                                          ("sinc3d", [40, 36, 30], [2, 3, 2], 2, [7, 6, 6], 1)]:
        f = ref.gen_field(gen, npts)
        rd = ref.RefDecomposition(npts, blocks, p, nc, ov)
        r = ref.solve(rd, f, max_outer_iterations=20, log_errors=False)
        dec = m.partition(npts, [(-4, 4)] * len(npts), blocks, p, nc, ov)
        g = m.solve(m.Field(npts, [(-4, 4)] * len(npts), f), dec,
                    m.SolverConfig(max_outer_iterations=20, log_errors=False))
        assert g.constraint_iterations == r.constraint_iterations
        assert close(g.model.controls, r.controls)
        assert abs(g.global_linf - r.global_linf) <= RTOL * max(1, r.global_linf)


def test_solve_enforce_off_and_determinism(ctx):
    cfg = SMALL["C5s"]
    values = W.make_field_numpy(cfg)
    g, o, s = run_both(cfg, values, enforce=False)
    assert_solve_parity(g, o)
    # bitwise run-to-run determinism of the whole solve
    s.run(values.reshape(-1))
    again = s.result()
    assert np.array_equal(again.model.controls, g.model.controls)
    assert again.global_l2 == g.global_l2


def test_device_resident_input(ctx):
    import torch
    cfg = SMALL["C3s"]
    values = W.make_field_numpy(cfg)
    dec = m.partition(cfg.grid, cfg.bounds, cfg.blocks, cfg.degree, cfg.nctrl, cfg.overlap)
    s = m.Solver(dec, m.SolverConfig(max_outer_iterations=20, log_errors=False))
    s.run(values.reshape(-1))
    host = s.result()
    t = torch.from_numpy(values).cuda().contiguous()
    s.run(t, on_device=True)
    dev = s.result()
    assert np.array_equal(host.model.controls, dev.model.controls)
    assert s.last_launches() > 0


def test_solve_host_e2e(ctx):
    cfg = SMALL["C2"]
    values = W.make_field_numpy(cfg)
    dec = m.partition(cfg.grid, cfg.bounds, cfg.blocks, cfg.degree, cfg.nctrl, cfg.overlap)
    s = m.Solver(dec, m.SolverConfig(max_outer_iterations=20, log_errors=False))
    out_c = np.zeros(tuple(dec.n_ctrl))
    out_e = np.zeros(cfg.grid)
    s.run_host(values, out_c, out_e)
    s.run(values.reshape(-1))
    r = s.result()
    assert np.array_equal(out_c, r.model.controls)
    assert np.array_equal(out_e, r.global_error)


@pytest.mark.parametrize("grid", [(200, 199), (41, 38, 37)])
def test_odd_extent_fallback_path(ctx, grid):
    """Odd last extent: field rows are not 16-B multiples, so the TMA passes
    are not eligible and the generic register-prefetch kernels run."""
    if len(grid) == 2:
        cfg = W.Config("odd2", grid, (2, 3), 3, (20, 14), 3, "sinc_radial")
    else:
        cfg = W.Config("odd3", grid, (2, 2, 2), 2, (7, 7, 6), 2, "sinc_radial")
    values = W.make_field_numpy(cfg)
    g, o, _ = run_both(cfg, values)
    assert_solve_parity(g, o)


def test_tma_and_generic_paths_agree(ctx, monkeypatch):
    cfg = SMALL["C5s"]
    values = W.make_field_numpy(cfg)
    g_tma, o, _ = run_both(cfg, values)
    monkeypatch.setenv("MFADD_NO_TMA", "1")
    g_gen, _, _ = run_both(cfg, values)
    assert_solve_parity(g_tma, o)
    assert_solve_parity(g_gen, o)
    # the TMA last-axis pass sums row segments then adds their carries, the
    # generic one sums rows in order: equal to rounding
    for bt, bg in zip(g_tma.blocks, g_gen.blocks):
        assert np.max(np.abs(bt.p - bg.p)) <= 1e-12 * max(1.0, np.max(np.abs(bg.p)))


@pytest.mark.parametrize("name", ["C2", "C5s"])
def test_twisted_solve2d_knob(ctx, monkeypatch, name):
    """MFADD_TWIST=1: the fused 2-D solve with two-sided (twisted) banded
    passes, another elimination order of lsq.cpp:59-60: same contract."""
    cfg = SMALL[name]
    values = W.make_field_numpy(cfg)
    g_plain, o, _ = run_both(cfg, values)
    monkeypatch.setenv("MFADD_TWIST", "1")
    g_tw, _, _ = run_both(cfg, values)
    assert_solve_parity(g_tw, o)
    for bt, bg in zip(g_tw.blocks, g_plain.blocks):
        assert np.max(np.abs(bt.p - bg.p)) <= 1e-11 * max(1.0, np.max(np.abs(bg.p)))


FUSE3D_CASES = {
    "C3s": SMALL["C3s"],
    "C4s": SMALL["C4s"],
    # odd held extents along every axis, long last axis (two row segments: the
    # carries of the last-axis contraction reach k_solve3d)
    "long2": W.Config("long2", (44, 46, 300), (2, 2, 2), 2, (7, 8, 41), 2, "sinc_radial"),
}


@pytest.mark.parametrize("env", [{}, {"MFADD_S3_SLAB": "2"}, {"MFADD_S3_SLAB": "2", "MFADD_S3_NL": "4"},
                                 {"MFADD_S3_SLAB": "4", "MFADD_NO_A0_SLAB": "1"}, {"MFADD_S3_NL": "4"},
                                 {"MFADD_NO_FUSE3D": "1"}],
                         ids=["default", "slab2", "slab2-nl4", "slab4-walkers", "nl4", "unfused"])
@pytest.mark.parametrize("name", list(FUSE3D_CASES))
def test_fused_3d_solve_forms(ctx, monkeypatch, name, env):
    """Every form of the 3-D fit's solve stage against the oracle: the whole
    block in one k_solve3d CTA, axis-0 slabs + k_axis0_slab or the strided
    walkers, one or four lines per thread, and the unfused passes
    (lsq.cpp:57-61 in any order of the commuting axis operators)."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    cfg = FUSE3D_CASES[name]
    values = W.make_field_numpy(cfg)
    g, o, _ = run_both(cfg, values)
    assert_solve_parity(g, o)


def test_graph_replay_matches_direct(ctx, monkeypatch):
    """The first solve on a field pointer runs direct launches, the second
    captures the whole solve into a CUDA graph, later ones replay it: all must
    be bitwise identical (and identical to the never-graphed path)."""
    cfg = SMALL["C2"]
    values = W.make_field_numpy(cfg)
    dec = m.partition(cfg.grid, cfg.bounds, cfg.blocks, cfg.degree, cfg.nctrl, cfg.overlap)
    s = m.Solver(dec, m.SolverConfig(max_outer_iterations=20, log_errors=False))
    res = []
    for _ in range(4):
        s.run(values.reshape(-1))
        res.append(s.result())
    monkeypatch.setenv("MFADD_NO_GRAPH", "1")
    s.run(values.reshape(-1))
    res.append(s.result())
    for r in res[1:]:
        assert np.array_equal(r.model.controls, res[0].model.controls)
        assert np.array_equal(r.global_error, res[0].global_error)
        assert [e.dp_max for e in r.epochs] == [e.dp_max for e in res[0].epochs]
        assert r.global_l2 == res[0].global_l2 and r.constraint_iterations == res[0].constraint_iterations


@pytest.mark.parametrize("name", ["C1", "C2", "C3s", "C4s", "C5s"])
def test_log_errors_block_residuals(ctx, name):
    """record_epoch with log_errors (solver.cpp:357-364): residual_error
    (lsq.cpp:66-85) of every block's held lattice over its input box, each
    epoch, vs the reference.  D >= 2 runs the one-pass form (epoch snapshots
    of the shared copies, every epoch's residuals after the loop): checked on
    the first solve (direct launches), the second (graph capture) and the
    third (graph replay)."""
    cfg = SMALL[name]
    values = W.make_field_numpy(cfg)
    dec = m.partition(cfg.grid, cfg.bounds, cfg.blocks, cfg.degree, cfg.nctrl, cfg.overlap)
    scfg = m.SolverConfig(max_outer_iterations=20, log_errors=True)
    o = orc.solve(orc.Decomposition(cfg.grid, cfg.blocks, cfg.degree, cfg.nctrl, cfg.overlap), values, 20, 1e-10,
                  log_errors=True)
    s = m.Solver(dec, scfg)
    first = None
    for rep in range(3):
        s.run(values.reshape(-1))
        r = s.result(want_blocks=False, want_error=False)
        assert len(r.epochs) == len(o.block_errors)
        for e, ob in zip(r.epochs, o.block_errors):
            got = np.array(e.block_errors)
            ref = np.asarray(ob).reshape(got.shape)
            assert np.all(np.abs(got - ref) <= 1e-10 * np.maximum(1.0, np.abs(ref))), (name, rep, e.iteration)
        errs = [np.array(e.block_errors) for e in r.epochs]
        if first is None:
            first = errs
        else:  # bitwise reproducible across direct launches / capture / replay
            assert all(np.array_equal(a, b) for a, b in zip(errs, first)), (name, rep)
    # the solve itself is unchanged by logging
    r2 = m.solve(m.Field(list(cfg.grid), list(cfg.bounds), values), dec,
                 m.SolverConfig(max_outer_iterations=20, log_errors=False))
    assert np.array_equal(r.model.controls, r2.model.controls)
    s.close()


def test_solve_host_batch_pipelined(ctx):
    """mfadd_solve_host_batch (overlapped H2D / solve / D2H over a stream of
    fields) returns exactly the results of one mfadd_solve_host per field."""
    cfg = SMALL["C5s"]
    dec = m.partition(cfg.grid, cfg.bounds, cfg.blocks, cfg.degree, cfg.nctrl, cfg.overlap)
    base = W.make_field_numpy(cfg)
    fields = [np.ascontiguousarray(base * (1.0 + 0.25 * k) + 0.01 * k) for k in range(5)]
    s = m.Solver(dec, m.SolverConfig(max_outer_iterations=20, log_errors=False))
    want = []
    for f in fields:
        c, e = np.zeros(tuple(dec.n_ctrl)), np.zeros(cfg.grid)
        s.run_host(f, c, e)
        want.append((c, e, s.summary.global_l2, s.summary.constraint_iterations))
    outs_c = [np.zeros(tuple(dec.n_ctrl)) for _ in fields]
    outs_e = [np.zeros(cfg.grid) for _ in fields]
    for _ in range(2):  # second pass replays the cached graphs of both slots
        sums = s.run_host_batch(fields, outs_c, outs_e)
        for (c, e, l2, it), oc, oe, sm in zip(want, outs_c, outs_e, sums):
            assert np.array_equal(oc, c) and np.array_equal(oe, e)
            assert sm.global_l2 == l2 and sm.constraint_iterations == it
    # the getters describe the last solve of the batch
    r = s.result(want_blocks=False)
    assert np.array_equal(r.model.controls, want[-1][0])
