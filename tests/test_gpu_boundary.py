"""Unit sub-boundaries of SURVEY §8(b) through the C ABI, checked against the
reference itself (oracle/_ref, the unmodified sources):

  residual_error   lsq.hpp:41, lsq.cpp:66-85   (pointwise bitwise, l2/linf)
  find_span        knots.hpp:36, knots.cpp:83-106 (bit-exact)
  basis_funs       knots.hpp:53, knots.cpp:108-129 (bit-exact, one-sided spans)
  basis_derivs     knots.hpp:56, knots.cpp:131-203 (bit-exact via eval_deriv)
  SingularFitError lsq.cpp:46-55 with uncovered_column lsq.cpp:25-35 (span equal)
and the solver's buffer checks (solver.cpp:335-338).
"""
import numpy as np
import pytest

import paper_2210_06528_b200 as m
from oracle import ref

pytestmark = pytest.mark.gpu

needs_ref = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")


def _kv(p, n, rng=None, repeated=False):
    kv = m.make_knot_vector(p, n)
    if rng is not None:  # strongly non-uniform interior knots (optionally a repeated one)
        inner = np.sort(rng.uniform(0, 1, n - p - 1))
        if repeated and len(inner) > 3:
            inner[2] = inner[1]
        kn = np.concatenate([np.zeros(p + 1), inner, np.ones(p + 1)])
        kv = m.KnotVector(p, kn)
    return kv


@needs_ref
@pytest.mark.parametrize("d", [1, 2, 3])
def test_residual_error_vs_reference(ctx, d):
    rng = np.random.default_rng(4100 + d)
    for p in (2, 3, 5):
        kvs, params, windows = [], [], []
        for k in range(d):
            n = p + 1 + int(rng.integers(4, 14))
            kv = m.make_knot_vector(p, n)
            lo = int(rng.integers(0, 3))
            hi = n - int(rng.integers(0, 3))
            # parameters over a sub-range: rows at the window edges are clipped
            u = np.sort(rng.uniform(0.05, 0.95, int(rng.integers(hi - lo + 2, hi - lo + 30))))
            kvs.append(kv)
            params.append(u)
            windows.append((lo, hi))
        q = rng.standard_normal(tuple(len(u) for u in params))
        P = rng.standard_normal(tuple(h - l for l, h in windows))
        lp = m.LocalProblem(kvs, params, windows, q)
        g = m.residual_error(lp, P, ctx=ctx)
        l2, linf, pw = ref.residual_error([k.knots for k in kvs], p, params, windows, q, P)
        assert np.array_equal(g.pointwise, pw), (d, p, np.abs(g.pointwise - pw).max())
        assert g.linf == linf
        assert abs(g.l2 - l2) <= 1e-13 * l2


@needs_ref
def test_residual_error_of_fit(ctx):
    # the fit's own residual: residual_error(problem, fit_unconstrained(problem))
    rng = np.random.default_rng(77)
    kvs = [m.make_knot_vector(3, 12), m.make_knot_vector(3, 10)]
    params = [np.linspace(0, 1, 40), np.linspace(0, 1, 33)]
    windows = [(0, 12), (0, 10)]
    q = rng.standard_normal((40, 33))
    lp = m.LocalProblem(kvs, params, windows, q)
    P = m.fit_unconstrained(lp, ctx)
    g = m.residual_error(lp, P, want_pointwise=False, ctx=ctx)
    Pr = ref.fit_unconstrained([k.knots for k in kvs], 3, params, windows, q)
    l2, linf, _ = ref.residual_error([k.knots for k in kvs], 3, params, windows, q, Pr)
    assert g.pointwise is None
    assert abs(g.l2 - l2) <= 1e-10 * l2 and abs(g.linf - linf) <= 1e-10 * linf


def test_residual_error_shape_checks(ctx):
    kv = m.make_knot_vector(3, 8)
    lp = m.LocalProblem([kv], [np.linspace(0, 1, 20)], [(0, 8)], np.zeros(20))
    with pytest.raises(m.InvalidArgument):
        m.residual_error(lp, np.zeros(7), ctx=ctx)


@needs_ref
def test_find_span_and_basis_funs_bit_exact(ctx):
    rng = np.random.default_rng(20240811)  # test_knots.cpp:78-112 seed
    for p in (1, 2, 3, 4, 5, 7):
        for trial in range(3):
            n = p + 1 + int(rng.integers(3, 25))
            kv = _kv(p, n, rng if trial else None, repeated=trial == 2)
            u = np.concatenate([rng.uniform(0, 1, 300), kv.knots[p:n + 1], [0.0, 1.0]])
            spans, vals = m.basis_funs_batch(kv, u, ctx=ctx)
            for i, x in enumerate(u):
                s = ref.find_span(kv.knots, p, float(x))
                assert spans[i] == s, (p, x)
                assert np.array_equal(vals[i, 0], ref.basis_funs(kv.knots, p, s, float(x)))
            assert m.find_span(kv, 0.37, ctx) == ref.find_span(kv.knots, p, 0.37)


@needs_ref
def test_basis_funs_one_sided_span(ctx):
    # basis_funs at the adjacent span with u on its boundary: the left piece
    kv = m.make_knot_vector(3, 10)
    for s in range(4, 10):
        u = float(kv.knots[s])
        b = m.basis_funs(kv, s - 1, u, ctx)
        assert b.span == s - 1
        assert np.array_equal(b.values, ref.basis_funs(kv.knots, 3, s - 1, u))
    with pytest.raises(m.InvalidArgument):
        m.basis_funs(kv, 1, 0.5, ctx)  # span < p
    with pytest.raises(m.OutOfRange):
        m.find_span(kv, 1.5, ctx)


@needs_ref
def test_basis_derivs_bit_exact_via_eval(ctx):
    # row k of basis_derivs = eval_deriv of the unit lattices e_j (the
    # reference's eval multiplies by 1.0 and adds to 0.0: exact)
    rng = np.random.default_rng(5)
    for p in (2, 3, 5):
        n = p + 8
        kv = _kv(p, n, rng)
        for x in rng.uniform(0, 1, 20):
            s = ref.find_span(kv.knots, p, float(x))
            b = m.basis_derivs(kv, s, float(x), p, ctx)
            assert np.array_equal(b.derivatives[0], b.values)
            for k in range(1, p + 1):
                for j in range(p + 1):
                    e = np.zeros(n)
                    e[s - p + j] = 1.0
                    r = ref.eval_points(e, [kv.knots], [p], np.array([[x]]), orders=[k])
                    assert b.deriv(k, j) == r[0], (p, k, j)
            assert abs(b.derivatives[1:].sum(axis=1)).max() < 1e-8 * max(1.0, abs(b.derivatives).max())
    with pytest.raises(m.InvalidArgument):
        m.basis_derivs(m.make_knot_vector(2, 5), 2, 0.1, 3, ctx)


@needs_ref
def test_singular_span_equals_reference(ctx):
    # test_lsq.cpp:191-215: SingularFitError{dim, span} exactly when the
    # reference throws it, with its uncovered column and message
    cases = [(2, 8, [0.3 * j / 10.0 for j in range(11)]),
             (3, 12, list(np.linspace(0.5, 1.0, 30))),
             (3, 12, list(np.linspace(0.0, 0.1, 15)) + list(np.linspace(0.9, 1.0, 15))),
             (3, 10, list(np.linspace(0.0, 0.2, 15)) + list(np.linspace(0.8, 1.0, 15)))]  # not singular
    raised = 0
    for p, n, params in cases:
        kv = m.make_knot_vector(p, n)
        lp = m.LocalProblem([kv], [np.array(params)], [(0, n)], np.ones(len(params)))
        try:
            ref.fit_unconstrained([kv.knots], p, [np.array(params)], [(0, n)], np.ones(len(params)))
            m.fit_unconstrained(lp, ctx)  # must not raise either
            continue
        except ref.RefError as er:
            assert er.code == 3
            with pytest.raises(m.SingularFitError) as ei:
                m.fit_unconstrained(lp, ctx)
            assert (ei.value.dim, ei.value.span) == (er.dim, er.span)
            assert str(ei.value) == str(er).split("] ", 1)[1]
            raised += 1
    assert raised == 3


def test_solver_buffer_checks(ctx):
    import torch
    dec = m.partition((64, 48), [(-1, 1), (-1, 1)], (2, 2), 3, (12, 10), 0)
    s = m.Solver(dec, m.SolverConfig(log_errors=False), ctx)
    good = torch.zeros((64, 48), dtype=torch.float64, device="cuda")
    s.run(good, on_device=True)
    with pytest.raises(m.InvalidArgument):
        s.run(torch.zeros((48, 64), dtype=torch.float64, device="cuda"), on_device=True)  # transposed extents
    with pytest.raises(m.InvalidArgument):
        s.run(torch.zeros((64, 48), dtype=torch.float32, device="cuda"), on_device=True)
    with pytest.raises(m.InvalidArgument):
        s.run(torch.zeros(64 * 48 - 1, dtype=torch.float64, device="cuda"), on_device=True)
    with pytest.raises(m.InvalidArgument):
        s.run(good.t(), on_device=True)  # non-contiguous
    with pytest.raises(m.InvalidArgument):
        s.run(np.zeros((48, 64)))
    hf = np.zeros((64, 48))
    with pytest.raises(m.InvalidArgument):
        s.run_host(hf, np.zeros(24 * 20 - 1))
    with pytest.raises(m.InvalidArgument):
        s.run_host(good, np.zeros(24 * 20))  # a device field on the host path
    s.close()
