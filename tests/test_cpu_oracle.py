"""Pin the C restatement oracle (oracle/liboracle.so) before trusting it:
against the golden fixtures generated from the reference implementation
(tests/golden/make_golden.py), against the reference library itself where it
is built (oracle/_ref), and against the reference unit tests' known answers
(test_knots.cpp, test_collocation.cpp, test_lsq.cpp, test_decode.cpp,
test_solver.cpp), re-expressed here."""
import glob
import hashlib
import os

import numpy as np
import pytest

from oracle import orc, ref
from paper_2210_06528_b200 import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def golden_values(g):
    if "values" in g:
        return g["values"]
    name, gen, grid, blocks, deg, nctrl, ov = [str(x) for x in g["cfg"]]
    cfg = W.Config(name, eval(grid), eval(blocks), int(deg), eval(nctrl), int(ov), gen)
    v = W.make_field_numpy(cfg)
    assert hashlib.sha256(np.ascontiguousarray(v).tobytes()).digest() == bytes(g["values_sha256"]), \
        "synthetic generator drifted from the golden fixture"
    return v


def solve_fixtures():
    return sorted(glob.glob(os.path.join(GOLD, "solve_*.npz")))


def test_collocation_golden():
    g = np.load(os.path.join(GOLD, "knots_collocation.npz"))
    for i in range(int(g["nkv"][0])):
        p, n, cl, cr = (int(x) for x in g[f"kv{i}_meta"])
        kn = orc.make_knot_vector(p, n, 0.0, 1.0, bool(cl), bool(cr))
        assert np.array_equal(kn, g[f"kv{i}_knots"])
        fc, cnt, vals = orc.collocation(kn, p, g[f"kv{i}_params"])
        assert np.array_equal(fc, g[f"kv{i}_fc"])
        assert np.array_equal(cnt, g[f"kv{i}_cnt"])
        assert np.array_equal(vals, g[f"kv{i}_vals"])  # bitwise: same operation order, no FMA


@pytest.mark.parametrize("path", solve_fixtures(), ids=lambda p: os.path.basename(p)[6:-4])
def test_solve_golden(path):
    g = np.load(path)
    values = golden_values(g)
    p, ov, clamp, iters = int(g["degree"][0]), int(g["overlap"][0]), bool(g["clamp"][0]), int(g["max_iters"][0])
    dec = orc.Decomposition(g["grid"].tolist(), g["blocks"].tolist(), p, g["nctrl"].tolist(), ov, clamp)
    assert np.array_equal(dec.blockdims(), g["blockdims"])
    bd = dec.blockdims()
    for b in (0, dec.nblocks - 1):
        for k in range(dec.rank):
            lo, hi = int(bd[b, k, 12]), int(bd[b, k, 13])
            u = np.array([j / (g["grid"][k] - 1) for j in range(lo, hi)])
            fc, cnt, vals = orc.collocation(dec.knots(k), p, u, int(bd[b, k, 8]), int(bd[b, k, 9]))
            assert np.array_equal(fc, g[f"rows_b{b}_d{k}_fc"])
            assert np.array_equal(cnt, g[f"rows_b{b}_d{k}_cnt"])
            assert np.array_equal(vals, g[f"rows_b{b}_d{k}_vals"])
    r = orc.solve(dec, values, iters, 1e-10, log_errors=True)
    conv, ci, fdp, l2, linf = g["scalars"]
    assert r.converged == bool(conv) and r.constraint_iterations == int(ci)
    # The oracle's Cholesky restates the reference's LLT call; both are built
    # with -ffp-contract=off, so agreement is bitwise here (tolerance 1e-13
    # guards only against toolchain drift).
    tol = 1e-13
    scale = max(1.0, float(np.abs(g["controls"]).max()))
    assert np.abs(r.controls - g["controls"]).max() <= tol * scale
    assert np.abs(r.epochs - g["epochs"]).max() <= tol * max(1.0, float(np.abs(g["epochs"]).max()))
    assert np.abs(r.final_jumps - g["final_jumps"]).max(initial=0) <= tol * scale
    assert abs(r.global_l2 - l2) <= tol * max(1, l2) and abs(r.global_linf - linf) <= tol * max(1, linf)
    stride = int(g["global_error_stride"][0])
    assert np.abs(r.global_error.reshape(-1)[::stride] - g["global_error"]).max() <= tol * scale
    for be_o, be_g in zip(r.block_errors, g["block_errors"]):
        assert np.abs(be_o - be_g).max() <= tol * max(1.0, float(np.abs(be_g).max()))
    assert np.abs(r.blocks_p[0] - g["block_p0"]).max() <= tol * scale
    assert np.abs(r.blocks_p[-1] - g["block_plast"]).max() <= tol * scale


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
def test_oracle_matches_reference_library_directly():
    rng = np.random.default_rng(77)
    for gen, npts, blocks, p, nc, ov in [("sinc2d", [50, 46], [2, 3], 4, [9, 8], 2),
                                          ("sinc1d-sym", [900], [3], 5, [20], 4),
                                          ("sinc2d", [60, 60], [3, 3], 3, [8, 8], 3),
                                          ("sinc3d", [30, 28, 26], [2, 2, 2], 3, [7, 7, 6], 1)]:
        f = ref.gen_field(gen, npts) + 0.01 * rng.standard_normal(npts)
        try:
            r = ref.solve(ref.RefDecomposition(npts, blocks, p, nc, ov), f, 20, 1e-10, log_errors=False)
        except ref.RefError as e:  # same exception, same message
            with pytest.raises(orc.OracleError) as oe:
                orc.solve(orc.Decomposition(npts, blocks, p, nc, ov), f, 20, 1e-10)
            assert (oe.value.code, str(oe.value)) == (e.code, str(e))
            continue
        o = orc.solve(orc.Decomposition(npts, blocks, p, nc, ov), f, 20, 1e-10)
        assert r.constraint_iterations == o.constraint_iterations
        assert np.array_equal(r.controls, o.controls)
        assert np.array_equal(r.epochs, o.epochs)


# ------------------------------------------------------------ known answers


def test_knots_known_answers():
    # test_knots.cpp:13-46
    assert orc.make_knot_vector(2, 3).tolist() == [0, 0, 0, 1, 1, 1]
    assert orc.make_knot_vector(3, 5).tolist() == [0, 0, 0, 0, 0.5, 1, 1, 1, 1]
    assert orc.make_knot_vector(2, 4, 0, 1, True, False).tolist() == [0, 0, 0, 0.5, 1, 1.5, 2]
    assert orc.make_knot_vector(2, 4, 0, 1, False, True).tolist() == [-1, -0.5, 0, 0.5, 1, 1, 1]
    with pytest.raises(orc.OracleError):
        orc.make_knot_vector(3, 3)
    kn = [0, 0, 0, 0.5, 1, 1, 1.0]
    assert orc.find_span(kn, 2, 0.25) == 2 and orc.find_span(kn, 2, 1.0) == 3 and orc.find_span(kn, 2, 0.5) == 3
    for u in (1.5, -0.1):
        with pytest.raises(orc.OracleError) as e:
            orc.find_span(kn, 2, u)
        assert e.value.code == 2
    v = orc.basis_funs([0, 0, 0, 1, 1, 1.0], 2, 2, 0.5)
    assert np.allclose(v, [0.25, 0.5, 0.25], rtol=0, atol=1e-14)


def test_partition_of_unity_sweep():
    # test_knots.cpp:78-112 (seed 20240811): rows sum to one
    rng = np.random.default_rng(20240811)
    for _ in range(200):
        p = int(rng.integers(1, 7))
        n = p + 1 + int(rng.integers(0, 12))
        kn = orc.make_knot_vector(p, n, 0, 1, bool(rng.integers(0, 2)), bool(rng.integers(0, 2)))
        u = rng.uniform(kn[p], kn[n])
        v = orc.basis_funs(kn, p, orc.find_span(kn, p, u), u)
        assert (v >= -1e-14).all() and abs(v.sum() - 1) < 1e-12


def test_lsq_dense_oracle():
    # test_lsq.cpp:131-146 (seed 5150): Kronecker solve == dense LSQ up to 12^d
    rng = np.random.default_rng(5150)
    for d in (1, 2, 3):
        kn = orc.make_knot_vector(2, 6)
        u = np.array([j / 11 for j in range(12)])
        q = rng.uniform(-1, 1, (12,) * d)
        P = orc.fit_unconstrained([kn] * d, 2, [u] * d, [(0, 6)] * d, q)
        fc, cnt, vals = orc.collocation(kn, 2, u)
        A1 = np.zeros((12, 6))
        for j in range(12):
            A1[j, fc[j]:fc[j] + cnt[j]] = vals[j, :cnt[j]]
        A = A1
        for _ in range(d - 1):
            A = np.kron(A, A1)
        sol = np.linalg.lstsq(A, q.reshape(-1), rcond=None)[0]
        assert np.abs(P.reshape(-1) - sol).max() < 1e-9


def test_singular_and_underdetermined():
    # test_lsq.cpp:191-215
    kn = orc.make_knot_vector(2, 8)
    with pytest.raises(orc.OracleError) as e:
        orc.fit_unconstrained([kn], 2, [np.array([0.3 * j / 10 for j in range(11)])], [(0, 8)], np.ones(11))
    assert e.value.code == 3 and e.value.dim == 0 and e.value.span >= 0
    with pytest.raises(orc.OracleError) as e:
        orc.fit_unconstrained([kn], 2, [np.linspace(0, 1, 5)], [(0, 8)], np.zeros(5))
    assert e.value.code == 1


def test_decode_brute_force():
    # test_decode.cpp:68-118 (seeds 7, 99): axis decode == brute tensor sum
    for seed, d in ((7, 2), (99, 3)):
        rng = np.random.default_rng(seed)
        kns = [orc.make_knot_vector(3, 6 + k) for k in range(d)]
        P = rng.standard_normal(tuple(6 + k for k in range(d)))
        params = [np.sort(rng.uniform(0, 1, 5)) for _ in range(d)]
        out = orc.decode(P, kns, 3, params)
        for idx in np.ndindex(*out.shape):
            bases = []
            for k in range(d):
                u = params[k][idx[k]]
                s = orc.find_span(kns[k], 3, u)
                row = np.zeros(len(kns[k]) - 4)
                row[s - 3:s + 1] = orc.basis_funs(kns[k], 3, s, u)
                bases.append(row)
            w = bases[0]
            for b in bases[1:]:
                w = np.multiply.outer(w, b)
            assert abs(float((w * P).sum()) - out[idx]) <= 1e-12


def test_solver_known_answers():
    if not ref.available():
        pytest.skip("reference generators live in oracle/_ref")
    # test_solver.cpp:169-187
    f = ref.gen_field("sinc1d-asym", [2000])
    r = orc.solve(orc.Decomposition([2000], [2], 3, [30], 3), f)
    assert r.converged and r.constraint_iterations == 1 and len(r.epochs) == 3
    assert r.epochs[0, 2] > 1e-12 and r.epochs[1, 2] < 1e-12 and r.epochs[2, 1] < 1e-10
    # test_solver.cpp:189-205
    f = ref.gen_field("sinc2d", [64, 64])
    r = orc.solve(orc.Decomposition([64, 64], [2, 2], 3, [12, 12], 0), f)
    assert r.constraint_iterations == 2 and len(r.epochs) == 4
    assert r.epochs[1, 3] > 1e-12 and r.epochs[2, 3] < 1e-12 and r.epochs[3, 1] < 1e-10
    # test_solver.cpp:301-310
    r = orc.solve(orc.Decomposition([64, 64], [2, 2], 3, [12, 12], 0), f, max_outer_iterations=1)
    assert not r.converged and r.constraint_iterations == 1 and r.final_dp >= 1e-10
