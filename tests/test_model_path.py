"""SURVEY §8(f) rows 2-4 against the reference itself (oracle/_ref, the
unmodified reference sources): the MfaModel output path (MFDD v1 container,
decode_grid, eval / eval_deriv), the continuity probe (eval_deriv_sided,
basis_derivs, continuity_jumps) and the raw-grid reader.

Bars: MFDD files byte-identical with the reference writer and read back
bit-exact (test_field_io.cpp:128-183); point evaluations and probe jumps
bitwise equal (explicit RN arithmetic in the reference's order); decode_grid
within 1e-12 relative (the grid decode contracts with FMA); raw grids
bit-exact; error types and messages as the reference's.
"""
import os

import numpy as np
import pytest

import paper_2210_06528_b200 as m
from oracle import ref

needs_ref = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")


def random_model(rank, degree, nctrl, seed, clamp=True):
    rng = np.random.default_rng(seed)
    kvs = [m.make_knot_vector(degree, n, 0.0, 1.0, clamp, clamp) for n in nctrl]
    ctrl = rng.standard_normal(tuple(nctrl))
    bounds = [(-1.5 - d, 2.0 + 0.5 * d) for d in range(rank)]
    return m.MfaModel([degree] * rank, kvs, ctrl, bounds, {"source": "sinc", "grid": "64x64", "a": "1"})


# ------------------------------------------------------------------ MFDD (host I/O, CPU suite)
@needs_ref
@pytest.mark.parametrize("rank,clamp", [(1, True), (2, True), (3, False)])
def test_mfdd_bytes_match_reference_writer(tmp_path, rank, clamp):
    mdl = random_model(rank, 3, [9, 7, 6][:rank], 20240811 + rank, clamp)
    ours, theirs = tmp_path / "ours.mfa", tmp_path / "ref.mfa"
    m.write_mfa(mdl, ours)
    ref.write_mfa(theirs, [k.knots for k in mdl.kvs], mdl.degrees, mdl.controls, [k.clamp_left for k in mdl.kvs],
                  [k.clamp_right for k in mdl.kvs], mdl.bounds, mdl.provenance)
    assert ours.read_bytes() == theirs.read_bytes()


@needs_ref
def test_mfdd_round_trip_bit_exact(tmp_path):
    mdl = random_model(2, 4, [11, 8], 5150, clamp=False)
    mdl.controls[0, 0] = -0.0
    mdl.controls[1, 2] = 1e-310  # subnormal survives
    p = tmp_path / "m.mfa"
    ref.write_mfa(p, [k.knots for k in mdl.kvs], mdl.degrees, mdl.controls, [k.clamp_left for k in mdl.kvs],
                  [k.clamp_right for k in mdl.kvs], mdl.bounds, mdl.provenance)
    back = m.read_mfa(p)
    assert back.degrees == mdl.degrees and back.bounds == mdl.bounds and back.provenance == mdl.provenance
    assert back.controls.tobytes() == np.ascontiguousarray(mdl.controls).tobytes()
    for a, b in zip(back.kvs, mdl.kvs):
        assert a.knots.tobytes() == b.knots.tobytes()
        assert (a.degree, a.clamp_left, a.clamp_right) == (b.degree, b.clamp_left, b.clamp_right)
    back.validate()
    # ours -> ours
    q = tmp_path / "n.mfa"
    m.write_mfa(back, q)
    assert q.read_bytes() == p.read_bytes()


@needs_ref
def test_mfdd_error_paths_match_reference(tmp_path):
    mdl = random_model(2, 3, [7, 7], 1)
    good = tmp_path / "g.mfa"
    m.write_mfa(mdl, good)
    raw = good.read_bytes()
    cases = {
        "magic": b"MFDX" + raw[4:],
        "version": raw[:4] + (2).to_bytes(4, "little") + raw[8:],
        "dims": raw[:8] + (4).to_bytes(4, "little") + raw[12:],
        "truncated": raw[:-5],
        "short": raw[:3],
    }
    for name, data in cases.items():
        p = tmp_path / f"{name}.mfa"
        p.write_bytes(data)
        code, msg = ref.read_mfa_status(p)
        assert code == 4, (name, code, msg)  # std::runtime_error
        with pytest.raises(m.RuntimeFault) as ei:
            m.read_mfa(p)
        assert str(ei.value).endswith(msg) or msg in str(ei.value), (name, str(ei.value), msg)
    code, msg = ref.read_mfa_status(tmp_path / "missing.mfa")
    with pytest.raises(m.RuntimeFault) as ei:
        m.read_mfa(tmp_path / "missing.mfa")
    assert msg in str(ei.value)


@needs_ref
def test_mfdd_write_validates_like_reference(tmp_path):
    mdl = random_model(2, 3, [7, 7], 2)
    bad = m.MfaModel(mdl.degrees, mdl.kvs, mdl.controls[:, :6], mdl.bounds)
    with pytest.raises(m.InvalidArgument, match="control extent must equal #knots - p - 1 in dimension 1"):
        m.write_mfa(bad, tmp_path / "x.mfa")
    with pytest.raises(ref.RefError, match="control extent must equal #knots - p - 1 in dimension 1"):
        ref.write_mfa(tmp_path / "y.mfa", [k.knots for k in bad.kvs], bad.degrees, bad.controls, [1, 1], [1, 1],
                      bad.bounds, {})


# ------------------------------------------------------------------ GPU rows
def _points(rng, kvs, npts, on_knots=0.3):
    """Random parameters, a share of them exactly on interior knots (the
    sided-span cases) and on the domain ends."""
    cols = []
    for kv in kvs:
        lo, hi = kv.domain_min(), kv.domain_max()
        u = rng.uniform(lo, hi, npts)
        inner = kv.knots[(kv.knots > lo) & (kv.knots < hi)]
        pick = rng.random(npts) < on_knots
        if inner.size:
            u[pick] = rng.choice(inner, int(pick.sum()))
        u[0], u[-1] = lo, hi
        cols.append(u)
    return np.stack(cols, 1)


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("rank,degree,clamp", [(1, 3, True), (2, 3, False), (2, 5, True), (3, 4, False)])
def test_eval_points_bitwise_vs_reference(ctx, rank, degree, clamp):
    rng = np.random.default_rng(77 + rank * 10 + degree)
    mdl = random_model(rank, degree, [degree + 9, degree + 6, degree + 4][:rank], 3 + degree, clamp)
    kl = [k.knots for k in mdl.kvs]
    pts = _points(rng, mdl.kvs, 257)
    for orders in (None, [0] * rank, [min(1, degree)] + [0] * (rank - 1), [degree] * rank,
                   [int(x) for x in rng.integers(0, degree + 1, rank)]):
        for side_dim, side in ((-1, 1), (0, m.Side.Below), (rank - 1, m.Side.Above), (rank - 1, m.Side.Below)):
            got = m.eval_points(mdl.controls, mdl.kvs, pts, orders, side_dim, side, ctx=ctx)
            exp = ref.eval_points(mdl.controls, kl, mdl.degrees, pts, orders, side_dim, side)
            assert got.tobytes() == exp.tobytes(), (orders, side_dim, side, np.abs(got - exp).max())


@pytest.mark.gpu
@needs_ref
def test_eval_windowed_col_offset_and_errors(ctx):
    mdl = random_model(2, 3, [14, 12], 11)
    kl = [k.knots for k in mdl.kvs]
    win = mdl.controls[3:11, 2:10].copy()  # a block's held window, col_offset (3, 2)
    rng = np.random.default_rng(9)
    # parameters whose active bases sit inside the window
    u0 = rng.uniform(mdl.kvs[0].knots[3 + 3 + 1], mdl.kvs[0].knots[11], 40)
    u1 = rng.uniform(mdl.kvs[1].knots[2 + 3 + 1], mdl.kvs[1].knots[10], 40)
    pts = np.stack([u0, u1], 1)
    got = m.eval_points(win, mdl.kvs, pts, [1, 2], ctx=ctx, col_offset=[3, 2])
    exp = ref.eval_points(win, kl, mdl.degrees, pts, [1, 2], col_offset=[3, 2])
    assert got.tobytes() == exp.tobytes()
    # the reference's failure modes, first failing point wins
    cases = [
        (dict(points=[[0.5, 0.5]], orders=[0, 4]), m.InvalidArgument, 1),
        (dict(points=[[0.5, 1.5]], orders=None), m.OutOfRange, 2),
        (dict(points=[[0.5, 0.5], [-0.1, 0.5]], orders=None), m.OutOfRange, 2),
    ]
    for kw, exc, code in cases:
        with pytest.raises(ref.RefError) as er:
            ref.eval_points(mdl.controls, kl, mdl.degrees, np.array(kw["points"]), kw["orders"])
        assert er.value.code == code
        with pytest.raises(exc) as eo:
            m.eval_points(mdl.controls, mdl.kvs, np.array(kw["points"]), kw["orders"], ctx=ctx)
        assert str(er.value).split("] ", 1)[1] in str(eo.value)
    with pytest.raises(ref.RefError) as er:  # window error
        ref.eval_points(win, kl, mdl.degrees, np.array([[0.01, 0.5]]), None, col_offset=[3, 2])
    with pytest.raises(m.OutOfRange, match="falls outside the control lattice window"):
        m.eval_points(win, mdl.kvs, np.array([[0.01, 0.5]]), None, col_offset=[3, 2], ctx=ctx)


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("rank,res", [(1, (1000,)), (2, (97, 130)), (3, (17, 23, 31))])
def test_decode_grid_vs_reference(ctx, rank, res):
    mdl = random_model(rank, 3, [20, 17, 12][:rank], 400 + rank)
    got = mdl.decode_grid(res, ctx=ctx)
    exp = ref.decode_grid(mdl.controls, [k.knots for k in mdl.kvs], mdl.degrees, res)
    scale = max(1.0, float(np.abs(exp).max()))
    assert float(np.abs(got - exp).max()) <= 1e-12 * scale
    with pytest.raises(m.InvalidArgument, match="need at least 2 points per dimension"):
        mdl.decode_grid((1,) + tuple(res[1:]), ctx=ctx)


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("rank", [1, 2, 3])
def test_continuity_jumps_model_bitwise(ctx, rank):
    mdl = random_model(rank, 4, [12, 10, 9][:rank], 600 + rank, clamp=False)
    kl = [k.knots for k in mdl.kvs]
    for dim in range(rank):
        u = float(mdl.kvs[dim].knots[4 + 3])  # an interior knot: a genuine interface
        for cs in (1, 5):
            got = m.continuity_jumps(mdl, dim, u, 3, cs, ctx=ctx)
            exp = ref.continuity_jumps_model(mdl.controls, kl, mdl.degrees, dim, u, 3, cs)
            assert np.array(got).tobytes() == exp.tobytes(), (dim, cs, got, exp)
    with pytest.raises(m.InvalidArgument, match="continuity_jumps: order exceeds degree"):
        m.continuity_jumps(mdl, 0, 0.5, 5, ctx=ctx)


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("grid,blocks,p,nctrl,ovl", [((400,), (4,), 3, (24,), 3), ((96, 80), (3, 2), 3, (20, 18), 3),
                                                     ((40, 36, 32), (2, 2, 2), 3, (12, 11, 10), 2)])
def test_solver_continuity_probe_vs_reference(ctx, grid, blocks, p, nctrl, ovl):
    """pipeline.cpp:210-228 on the solved block models: our held lattices agree
    with the reference's to rounding, so the jumps agree to 1e-9 of the field
    scale (and are ~0 at orders < p-? after convergence)."""
    rng = np.random.default_rng(31)
    vals = np.sin(np.linspace(0, 6, int(np.prod(grid)))).reshape(grid) + 0.1 * rng.standard_normal(grid)
    dec = m.partition(grid, [(0.0, 1.0)] * len(grid), blocks, p, nctrl, ovl)
    s = m.Solver(dec, m.SolverConfig(max_outer_iterations=20, tolerance=1e-10, log_errors=False, store_error=False),
                 ctx=ctx)
    s.run(vals.reshape(-1))
    order, got = s.continuity_probe(-1, 5)
    rd = ref.RefDecomposition(grid, blocks, p, nctrl, ovl)
    rorder, exp = ref.solve_and_probe(rd, vals, 20, 1e-10, -1, 5)
    assert order == rorder == p - 1
    scale = max(1.0, float(np.abs(vals).max()))
    assert np.allclose(got, exp, rtol=1e-6, atol=1e-9 * scale), (got, exp)


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("type_,order", [(0, 0), (0, 1), (1, 0), (1, 1)])
def test_read_raw_grid_bitwise(ctx, tmp_path, type_, order):
    rng = np.random.default_rng(type_ * 2 + order)
    dims = (13, 7, 5)
    v = rng.standard_normal(dims) * 1e3
    v.flat[0] = -0.0
    v.flat[1] = np.inf
    dt = np.dtype(np.float32 if type_ == 0 else np.float64).newbyteorder("<" if order == 0 else ">")
    p = tmp_path / "g.raw"
    v.astype(dt).tofile(p)
    fld = m.read_raw_grid(p, dims, type_, order, ctx=ctx)
    exp = ref.read_raw_grid(p, dims, type_, order)
    assert fld.values.tobytes() == exp.tobytes()
    assert fld.name == "g.raw" and fld.bounds == [(0.0, 1.0)] * 3
    # device destination (the field stays in HBM)
    import torch
    t = torch.empty(int(np.prod(dims)), dtype=torch.float64, device="cuda")
    m.read_raw_grid(p, dims, type_, order, device_out=t.data_ptr(), ctx=ctx)
    assert t.cpu().numpy().tobytes() == exp.reshape(-1).tobytes()
    # size mismatch: same error type and text
    with pytest.raises(ref.RefError) as er:
        ref.read_raw_grid(p, (13, 7, 6), type_, order)
    with pytest.raises(m.RuntimeFault) as eo:
        m.read_raw_grid(p, (13, 7, 6), type_, order, ctx=ctx)
    assert str(er.value).split("] ", 1)[1] in str(eo.value)
