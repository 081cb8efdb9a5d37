"""ctypes binding of oracle/_ref/libmfadd_ref.so — the UNMODIFIED reference
library (`/root/reference/proj/core/src/*.cpp`) plus oracle/ref_driver.cpp.

TEST INFRASTRUCTURE ONLY.  Importers allowed: tests/, __graft_entry__.smoke()
and bench.py's reference / cpu_baseline legs.  The product package never
imports anything under oracle/.

The library is built here (where /root/reference exists) by `make -C oracle
ref` and travels to the GPU box as a prebuilt file; on the box nothing reads
/root/reference.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libmfadd_ref.so")

_dp = C.POINTER(C.c_double)
_lp = C.POINTER(C.c_longlong)
_ip = C.POINTER(C.c_int)

_lib = None


class RefError(RuntimeError):
    """Raised for a non-zero status; `code` mirrors the reference exception type:
    1 invalid_argument, 2 out_of_range, 3 SingularFitError, 4 runtime_error,
    5 logic_error, 9 other."""

    def __init__(self, code, msg, dim=-1, span=-1):
        super().__init__(f"[{code}] {msg}")
        self.code, self.dim, self.span = code, dim, span


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{LIB_PATH} not built (make -C oracle ref)")
        L = C.CDLL(LIB_PATH, mode=C.RTLD_LOCAL)
        L.ref_last_error.restype = C.c_char_p
        L.ref_last_error_span.restype = C.c_longlong
        L.ref_dec_compression_ratio.restype = C.c_double
        L.ref_result_block_size.restype = C.c_longlong
        L.ref_dec_free.argtypes = [C.c_void_p]
        L.ref_result_free.argtypes = [C.c_void_p]
        for n in ("ref_dec_nblocks", "ref_dec_rank", "ref_dec_any_shared", "ref_dec_compression_ratio"):
            getattr(L, n).argtypes = [C.c_void_p]
        for n in ("ref_dec_blockdims", "ref_dec_coords", "ref_dec_nctrl", "ref_dec_exchange_volume",
                  "ref_dec_neighbors", "ref_dec_knots", "ref_dec_holder_ranges", "ref_dec_n_s",
                  "ref_dec_holders", "ref_result_scalars", "ref_result_epochs", "ref_result_block_errors",
                  "ref_result_final_jumps", "ref_result_controls", "ref_result_error",
                  "ref_result_block_size", "ref_result_block_p"):
            getattr(L, n).argtypes = None
        _lib = L
    return _lib


def _ptr(a, t):
    return a.ctypes.data_as(t)


def _check(rc):
    if rc != 0:
        L = lib()
        raise RefError(rc, L.ref_last_error().decode(), L.ref_last_error_dim(), L.ref_last_error_span())


# ---------------------------------------------------------------- knots
def make_knot_vector(degree, basis_count, a=0.0, b=1.0, clamp_left=True, clamp_right=True):
    out = np.zeros(basis_count + degree + 1 + 8, np.float64)
    n = C.c_int()
    _check(lib().ref_make_knot_vector(degree, basis_count, C.c_double(a), C.c_double(b), int(clamp_left),
                                      int(clamp_right), _ptr(out, _dp), len(out), C.byref(n)))
    return out[: n.value].copy()


def find_span(knots, degree, u):
    k = np.ascontiguousarray(knots, np.float64)
    s = C.c_int()
    _check(lib().ref_find_span(_ptr(k, _dp), len(k), degree, C.c_double(u), C.byref(s)))
    return s.value


def basis_funs(knots, degree, span, u):
    k = np.ascontiguousarray(knots, np.float64)
    out = np.zeros(degree + 1, np.float64)
    _check(lib().ref_basis_funs(_ptr(k, _dp), len(k), degree, span, C.c_double(u), _ptr(out, _dp)))
    return out


def collocation(knots, degree, params, col_lo=0, col_hi=None):
    k = np.ascontiguousarray(knots, np.float64)
    p = np.ascontiguousarray(params, np.float64)
    if col_hi is None:
        col_hi = len(k) - degree - 1
    m = len(p)
    fc = np.zeros(m, np.int64)
    cnt = np.zeros(m, np.int32)
    vals = np.zeros((m, degree + 1), np.float64)
    _check(lib().ref_collocation(_ptr(k, _dp), len(k), degree, _ptr(p, _dp), C.c_longlong(m),
                                 C.c_longlong(col_lo), C.c_longlong(col_hi), _ptr(fc, _lp), _ptr(cnt, _ip),
                                 _ptr(vals, _dp)))
    return fc, cnt, vals


# ---------------------------------------------------------------- lsq / decode
def _pack(knots_list, params_list):
    kn = np.concatenate([np.asarray(k, np.float64) for k in knots_list])
    ko = np.cumsum([0] + [len(k) for k in knots_list]).astype(np.int64)
    pm = np.concatenate([np.asarray(p, np.float64) for p in params_list])
    po = np.cumsum([0] + [len(p) for p in params_list]).astype(np.int64)
    return kn, ko, pm, po


def fit_unconstrained(knots_list, degree, params_list, windows, q):
    """fit_unconstrained (lsq.cpp:39-64) on one LocalProblem."""
    kn, ko, pm, po = _pack(knots_list, params_list)
    lo = np.array([w[0] for w in windows], np.int64)
    hi = np.array([w[1] for w in windows], np.int64)
    qq = np.ascontiguousarray(q, np.float64)
    out = np.zeros(tuple(int(h - l) for l, h in zip(lo, hi)), np.float64)
    _check(lib().ref_fit_unconstrained(len(knots_list), degree, _ptr(kn, _dp), _ptr(ko, _lp), _ptr(pm, _dp),
                                       _ptr(po, _lp), _ptr(lo, _lp), _ptr(hi, _lp), _ptr(qq, _dp),
                                       _ptr(out, _dp)))
    return out


def residual_error(knots_list, degree, params_list, windows, q, p):
    kn, ko, pm, po = _pack(knots_list, params_list)
    lo = np.array([w[0] for w in windows], np.int64)
    hi = np.array([w[1] for w in windows], np.int64)
    qq = np.ascontiguousarray(q, np.float64)
    pp = np.ascontiguousarray(p, np.float64)
    l2, linf = C.c_double(), C.c_double()
    pw = np.zeros_like(qq)
    _check(lib().ref_residual_error(len(knots_list), degree, _ptr(kn, _dp), _ptr(ko, _lp), _ptr(pm, _dp),
                                    _ptr(po, _lp), _ptr(lo, _lp), _ptr(hi, _lp), _ptr(qq, _dp), _ptr(pp, _dp),
                                    C.byref(l2), C.byref(linf), _ptr(pw, _dp)))
    return l2.value, linf.value, pw


def decode(controls, knots_list, degree, params_list, col_offset=None):
    kn, ko, pm, po = _pack(knots_list, params_list)
    c = np.ascontiguousarray(controls, np.float64)
    ext = np.array(c.shape, np.int64)
    off = None if col_offset is None else np.array(col_offset, np.int64)
    out = np.zeros(tuple(len(p) for p in params_list), np.float64)
    _check(lib().ref_decode(len(knots_list), degree, _ptr(kn, _dp), _ptr(ko, _lp), _ptr(pm, _dp), _ptr(po, _lp),
                            _ptr(ext, _lp), None if off is None else _ptr(off, _lp), _ptr(c, _dp),
                            _ptr(out, _dp)))
    return out


def gen_field(generator, npts):
    n = np.array(npts, np.int64)
    out = np.zeros(tuple(npts), np.float64)
    _check(lib().ref_gen_field(generator.encode(), len(npts), _ptr(n, _lp), _ptr(out, _dp)))
    return out


# ---------------------------------------------------------------- layout
BLOCKDIM_FIELDS = ("span_lo", "span_hi", "delta_lo", "delta_hi", "overlap_lo", "overlap_hi", "local_span_lo",
                   "local_span_hi", "dof_lo", "dof_hi", "own_lo", "own_hi", "input_lo", "input_hi",
                   "own_input_lo", "own_input_hi")


class RefDecomposition:
    """mfadd::partition (layout.cpp:217-342) result held by the reference."""

    def __init__(self, grid_dims, blocks_per_dim, degree, nctrl_per_block, overlap, clamp_interfaces=False,
                 bounds=None):
        rank = len(grid_dims)
        g = np.array(grid_dims, np.int64)
        b = np.array(blocks_per_dim, np.int32)
        nc = np.array(nctrl_per_block, np.int64)
        bd = None if bounds is None else np.array(bounds, np.float64).reshape(-1)
        h = C.c_void_p()
        _check(lib().ref_partition(rank, _ptr(g, _lp), None if bd is None else _ptr(bd, _dp), _ptr(b, _ip), degree,
                                   _ptr(nc, _lp), C.c_longlong(overlap), int(clamp_interfaces), C.byref(h)))
        self._h = h
        self.rank = rank
        self.degree = degree
        self.grid_dims = tuple(int(x) for x in grid_dims)
        self.bounds = bounds
        self.nblocks = lib().ref_dec_nblocks(h)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.ref_dec_free(self._h)
            self._h = None

    def blockdims(self):
        out = np.zeros((self.nblocks, self.rank, 16), np.int64)
        lib().ref_dec_blockdims(self._h, _ptr(out, _lp))
        return out

    def coords(self):
        out = np.zeros((self.nblocks, self.rank), np.int32)
        lib().ref_dec_coords(self._h, _ptr(out, _ip))
        return out

    def neighbors(self, block):
        buf = np.zeros(64, np.int32)
        n = lib().ref_dec_neighbors(self._h, block, _ptr(buf, _ip), 64)
        return buf[:n].tolist()

    def nctrl(self):
        out = np.zeros(self.rank, np.int64)
        lib().ref_dec_nctrl(self._h, _ptr(out, _lp))
        return out

    def knots(self, dim):
        buf = np.zeros(1 << 20, np.float64)
        n = lib().ref_dec_knots(self._h, dim, _ptr(buf, _dp), len(buf))
        return buf[:n].copy()

    def holder_ranges(self, dim):
        out = np.zeros((int(self.nctrl()[dim]), 2), np.int32)
        lib().ref_dec_holder_ranges(self._h, dim, _ptr(out, _ip))
        return out

    def n_s(self, dof):
        d = np.array(dof, np.int64)
        return lib().ref_dec_n_s(self._h, _ptr(d, _lp))

    def holders(self, dof):
        d = np.array(dof, np.int64)
        buf = np.zeros(16, np.int32)
        n = lib().ref_dec_holders(self._h, _ptr(d, _lp), _ptr(buf, _ip), 16)
        return buf[:n].tolist()

    def exchange_volume(self):
        out = np.zeros(self.nblocks, np.int64)
        lib().ref_dec_exchange_volume(self._h, _ptr(out, _lp))
        return out

    def compression_ratio(self):
        return lib().ref_dec_compression_ratio(self._h)

    def any_shared(self):
        return bool(lib().ref_dec_any_shared(self._h))


@dataclass
class RefSolveResult:
    converged: bool
    constraint_iterations: int
    final_dp: float
    global_l2: float
    global_linf: float
    epochs: np.ndarray  # (E, 4): iteration, dp_max, jump_ss, jump_ms
    final_jumps: np.ndarray  # (J, 4): a, b, linf_ss, linf_ms
    controls: np.ndarray
    global_error: np.ndarray
    blocks_p: list
    timings: dict = field(default_factory=dict)
    block_errors: list = field(default_factory=list)


def solve(dec: RefDecomposition, values, max_outer_iterations=10, tolerance=1e-10, workers=1, log_errors=True,
          enforce_continuity=True, want_blocks=True):
    """mfadd::solve (solver.cpp:332-440) on the reference library."""
    v = np.ascontiguousarray(values, np.float64)
    assert v.shape == dec.grid_dims, (v.shape, dec.grid_dims)
    bd = None if dec.bounds is None else np.array(dec.bounds, np.float64).reshape(-1)
    h = C.c_void_p()
    L = lib()
    _check(L.ref_solve(dec._h, _ptr(v, _dp), None if bd is None else _ptr(bd, _dp), max_outer_iterations,
                       C.c_double(tolerance), workers, int(log_errors), int(enforce_continuity), C.byref(h)))
    try:
        ints = np.zeros(4, np.int32)
        dbl = np.zeros(8, np.float64)
        L.ref_result_scalars(h, _ptr(ints, _ip), _ptr(dbl, _dp))
        L.ref_last_solve_seconds.restype = C.c_double
        solve_s = float(L.ref_last_solve_seconds())
        ep = np.zeros((int(ints[2]), 4), np.float64)
        L.ref_result_epochs(h, _ptr(ep, _dp))
        fj = np.zeros((int(ints[3]), 4), np.float64)
        L.ref_result_final_jumps(h, _ptr(fj, _dp))
        ctrl = np.zeros(tuple(int(x) for x in dec.nctrl()), np.float64)
        L.ref_result_controls(h, _ptr(ctrl, _dp))
        err = np.zeros(dec.grid_dims, np.float64)
        L.ref_result_error(h, _ptr(err, _dp))
        blocks = []
        if want_blocks:
            bdims = dec.blockdims()
            for b in range(dec.nblocks):
                shape = tuple(int(bdims[b, d, 9] - bdims[b, d, 8]) for d in range(dec.rank))
                pb = np.zeros(shape, np.float64)
                L.ref_result_block_p(h, b, _ptr(pb, _dp))
                blocks.append(pb)
        berr = []
        if log_errors:
            for e in range(int(ints[2])):
                buf = np.zeros((dec.nblocks, 2), np.float64)
                L.ref_result_block_errors(h, e, _ptr(buf, _dp))
                berr.append(buf)
        return RefSolveResult(bool(ints[0]), int(ints[1]), float(dbl[0]), float(dbl[1]), float(dbl[2]), ep, fj,
                              ctrl, err, blocks,
                              dict(setup=dbl[3], local_solve=dbl[4], exchange=dbl[5], constraint=dbl[6],
                                   decode=dbl[7], solve_s=solve_s), berr)
    finally:
        L.ref_result_free(h)


# ---------------------------------------------------------------- §8(f): model path, probe, raw grid
def _model_arrays(knots_list, degrees, controls):
    kn = np.ascontiguousarray(np.concatenate([np.asarray(k, np.float64) for k in knots_list]))
    ko = np.cumsum([0] + [len(k) for k in knots_list]).astype(np.int64)
    deg = np.array(degrees, np.int32)
    c = np.ascontiguousarray(controls, np.float64)
    ext = np.array(c.shape, np.int64)
    return kn, ko, deg, c, ext


def eval_points(controls, knots_list, degrees, points, orders=None, side_dim=-1, side=1, col_offset=None):
    """eval_deriv / eval_deriv_sided (decode.hpp:28-40), one reference call per point."""
    kn, ko, deg, c, ext = _model_arrays(knots_list, degrees, controls)
    pts = np.ascontiguousarray(np.atleast_2d(np.asarray(points, np.float64)))
    ords = None if orders is None else np.array(orders, np.int32)
    off = None if col_offset is None else np.array(col_offset, np.int64)
    out = np.zeros(pts.shape[0], np.float64)
    L = lib()
    L.ref_eval_points.argtypes = None
    _check(L.ref_eval_points(len(knots_list), _ptr(deg, _ip), _ptr(kn, _dp), _ptr(ko, _lp), _ptr(ext, _lp),
                             None if off is None else _ptr(off, _lp), _ptr(c, _dp), C.c_longlong(pts.shape[0]),
                             _ptr(pts, _dp), None if ords is None else _ptr(ords, _ip), side_dim, side,
                             _ptr(out, _dp)))
    return out


def decode_grid(controls, knots_list, degrees, res):
    """MfaModel::decode_grid (model.cpp:39-49)."""
    kn, ko, deg, c, ext = _model_arrays(knots_list, degrees, controls)
    r = np.array(res, np.int64)
    out = np.zeros(tuple(int(x) for x in res), np.float64)
    _check(lib().ref_decode_grid(len(knots_list), _ptr(deg, _ip), _ptr(kn, _dp), _ptr(ko, _lp), _ptr(ext, _lp),
                                 _ptr(c, _dp), _ptr(r, _lp), _ptr(out, _dp)))
    return out


def write_mfa(path, knots_list, degrees, controls, clamp_left, clamp_right, bounds, provenance):
    """write_mfa (model.cpp:93-118)."""
    kn, ko, deg, c, ext = _model_arrays(knots_list, degrees, controls)
    cl = np.array([int(x) for x in clamp_left], np.int32)
    cr = np.array([int(x) for x in clamp_right], np.int32)
    b = np.ascontiguousarray(np.array(bounds, np.float64).reshape(-1))
    keys = [str(k).encode() for k in provenance]
    vals = [str(provenance[k]).encode() for k in provenance]
    karr = (C.c_char_p * max(len(keys), 1))(*keys)
    varr = (C.c_char_p * max(len(vals), 1))(*vals)
    _check(lib().ref_write_mfa(str(path).encode(), len(knots_list), _ptr(deg, _ip), _ptr(cl, _ip), _ptr(cr, _ip),
                               _ptr(kn, _dp), _ptr(ko, _lp), _ptr(ext, _lp), _ptr(b, _dp), len(keys), karr, varr,
                               _ptr(c, _dp)))


def read_mfa_status(path):
    """(code, message) of read_mfa (model.cpp:120-167) on `path`; code 0 = ok."""
    L = lib()
    rc = L.ref_read_mfa_check(str(path).encode())
    return rc, (L.ref_last_error().decode() if rc else "")


def read_raw_grid(path, dims, type_, order):
    """read_raw_grid (field.cpp:149-191): type_ 0 f32 / 1 f64, order 0 little / 1 big."""
    d = np.array(dims, np.int64)
    out = np.zeros(tuple(int(x) for x in dims), np.float64)
    _check(lib().ref_read_raw_grid(str(path).encode(), len(dims), _ptr(d, _lp), type_, order, _ptr(out, _dp)))
    return out


def continuity_jumps_model(controls, knots_list, degrees, dim, u, max_order, cross_samples=5):
    """continuity_jumps(const MfaModel&, ...) (solver.cpp:244-261)."""
    kn, ko, deg, c, ext = _model_arrays(knots_list, degrees, controls)
    out = np.zeros(max_order + 1, np.float64)
    _check(lib().ref_continuity_jumps_model(len(knots_list), _ptr(deg, _ip), _ptr(kn, _dp), _ptr(ko, _lp),
                                            _ptr(ext, _lp), _ptr(c, _dp), dim, C.c_double(u), max_order,
                                            cross_samples, _ptr(out, _dp)))
    return out


def solve_and_probe(dec: "RefDecomposition", values, max_outer_iterations=20, tolerance=1e-10, probe_order=-1,
                    cross_samples=5):
    """solve() then the pipeline's continuity probe (pipeline.cpp:210-228,
    restated loop over continuity_jumps(BlockState, BlockState, ...))."""
    v = np.ascontiguousarray(values, np.float64)
    h = C.c_void_p()
    L = lib()
    L.ref_dec_span_param.restype = C.c_double
    L.ref_dec_span_param.argtypes = [C.c_void_p, C.c_int, C.c_longlong]
    _check(L.ref_solve(dec._h, _ptr(v, _dp), None, max_outer_iterations, C.c_double(tolerance), 1, 0, 1,
                       C.byref(h)))
    try:
        order = probe_order if probe_order >= 0 else dec.degree - 1
        jumps = np.zeros(order + 1, np.float64)
        coords = dec.coords()
        bdims = dec.blockdims()
        bpd = [int(coords[:, k].max()) + 1 for k in range(dec.rank)]
        buf = np.zeros(order + 1, np.float64)
        for b in range(dec.nblocks):
            for dim in range(dec.rank):
                if coords[b, dim] + 1 >= bpd[dim]:
                    continue
                ac = list(coords[b])
                ac[dim] += 1
                above = 0
                for k in range(dec.rank):
                    above = above * bpd[k] + int(ac[k])
                u = L.ref_dec_span_param(dec._h, dim, int(bdims[b, dim, 1]))
                _check(L.ref_continuity_jumps_blocks(dec._h, h, b, above, dim, C.c_double(u), order, cross_samples,
                                                     _ptr(buf, _dp)))
                jumps = np.maximum(jumps, buf)
        return order, jumps
    finally:
        L.ref_result_free(h)
