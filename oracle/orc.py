"""ctypes binding of oracle/liboracle.so — the plain-C restatement
(oracle/mfa_oracle.c) of the reference MFA encode path.

TEST INFRASTRUCTURE ONLY: importable from tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline leg; never from the product package.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle.so")

_dp = C.POINTER(C.c_double)
_lp = C.POINTER(C.c_int64)
_ip = C.POINTER(C.c_int)
_lib = None


class OracleError(RuntimeError):
    def __init__(self, code, msg, dim=-1, span=-1):
        super().__init__(f"[{code}] {msg}")
        self.code, self.dim, self.span = code, dim, span


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FileNotFoundError(f"{LIB_PATH} not built (make -C oracle oracle)")
        L = C.CDLL(LIB_PATH, mode=C.RTLD_LOCAL)
        L.orc_last_error.restype = C.c_char_p
        L.orc_last_error_span.restype = C.c_int64
        L.orc_dec_free.argtypes = [C.c_void_p]
        L.orc_result_free.argtypes = [C.c_void_p]
        L.orc_dec_nblocks.argtypes = [C.c_void_p]
        L.orc_basis_funs.argtypes = [_dp, C.c_int, C.c_int, C.c_double, _dp]
        _lib = L
    return _lib


def _ptr(a, t):
    return a.ctypes.data_as(t)


def _check(rc):
    if rc != 0:
        L = lib()
        raise OracleError(rc, L.orc_last_error().decode(), L.orc_last_error_dim(), L.orc_last_error_span())


def make_knot_vector(degree, basis_count, a=0.0, b=1.0, clamp_left=True, clamp_right=True):
    out = np.zeros(basis_count + degree + 1, np.float64)
    _check(lib().orc_make_knot_vector(degree, basis_count, C.c_double(a), C.c_double(b), int(clamp_left),
                                      int(clamp_right), _ptr(out, _dp)))
    return out


def find_span(knots, degree, u):
    k = np.ascontiguousarray(knots, np.float64)
    s = C.c_int()
    _check(lib().orc_find_span(_ptr(k, _dp), len(k), degree, C.c_double(u), C.byref(s)))
    return s.value


def basis_funs(knots, degree, span, u):
    k = np.ascontiguousarray(knots, np.float64)
    out = np.zeros(degree + 1, np.float64)
    lib().orc_basis_funs(_ptr(k, _dp), degree, span, u, _ptr(out, _dp))
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
    _check(lib().orc_collocation(_ptr(k, _dp), len(k), degree, _ptr(p, _dp), C.c_int64(m), C.c_int64(col_lo),
                                 C.c_int64(col_hi), _ptr(fc, _lp), _ptr(cnt, _ip), _ptr(vals, _dp)))
    return fc, cnt, vals


def _pack(knots_list, params_list):
    kn = np.concatenate([np.asarray(k, np.float64) for k in knots_list])
    ko = np.cumsum([0] + [len(k) for k in knots_list]).astype(np.int64)
    pm = np.concatenate([np.asarray(p, np.float64) for p in params_list])
    po = np.cumsum([0] + [len(p) for p in params_list]).astype(np.int64)
    return kn, ko, pm, po


def fit_unconstrained(knots_list, degree, params_list, windows, q):
    kn, ko, pm, po = _pack(knots_list, params_list)
    lo = np.array([w[0] for w in windows], np.int64)
    hi = np.array([w[1] for w in windows], np.int64)
    qq = np.ascontiguousarray(q, np.float64)
    out = np.zeros(tuple(int(h - l) for l, h in zip(lo, hi)), np.float64)
    _check(lib().orc_fit_unconstrained(len(knots_list), degree, _ptr(kn, _dp), _ptr(ko, _lp), _ptr(pm, _dp),
                                       _ptr(po, _lp), _ptr(lo, _lp), _ptr(hi, _lp), _ptr(qq, _dp),
                                       _ptr(out, _dp)))
    return out


def decode(controls, knots_list, degree, params_list, col_offset=None):
    kn, ko, pm, po = _pack(knots_list, params_list)
    c = np.ascontiguousarray(controls, np.float64)
    ext = np.array(c.shape, np.int64)
    off = None if col_offset is None else np.array(col_offset, np.int64)
    out = np.zeros(tuple(len(p) for p in params_list), np.float64)
    _check(lib().orc_decode(len(knots_list), degree, _ptr(kn, _dp), _ptr(ko, _lp), _ptr(pm, _dp), _ptr(po, _lp),
                            _ptr(ext, _lp), None if off is None else _ptr(off, _lp), _ptr(c, _dp),
                            _ptr(out, _dp)))
    return out


class Decomposition:
    """partition() restated (layout.cpp:217-342)."""

    def __init__(self, grid_dims, blocks_per_dim, degree, nctrl_per_block, overlap, clamp_interfaces=False):
        self.rank = len(grid_dims)
        self.degree = degree
        self.grid_dims = tuple(int(x) for x in grid_dims)
        g = np.array(grid_dims, np.int64)
        b = np.array(blocks_per_dim, np.int32)
        nc = np.array(nctrl_per_block, np.int64)
        h = C.c_void_p()
        _check(lib().orc_partition(self.rank, _ptr(g, _lp), _ptr(b, _ip), degree, _ptr(nc, _lp),
                                   C.c_int64(overlap), int(clamp_interfaces), C.byref(h)))
        self._h = h
        self.nblocks = lib().orc_dec_nblocks(h)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.orc_dec_free(self._h)
            self._h = None

    def blockdims(self):
        out = np.zeros((self.nblocks, self.rank, 16), np.int64)
        lib().orc_dec_blockdims(self._h, _ptr(out, _lp))
        return out

    def coords(self):
        out = np.zeros((self.nblocks, self.rank), np.int32)
        lib().orc_dec_coords(self._h, _ptr(out, _ip))
        return out

    def nctrl(self):
        out = np.zeros(self.rank, np.int64)
        lib().orc_dec_nctrl(self._h, _ptr(out, _lp))
        return out

    def knots(self, dim):
        n = lib().orc_dec_knots(self._h, dim, None)
        out = np.zeros(n, np.float64)
        lib().orc_dec_knots(self._h, dim, _ptr(out, _dp))
        return out

    def holder_ranges(self, dim):
        out = np.zeros((int(self.nctrl()[dim]), 2), np.int32)
        lib().orc_dec_holder_ranges(self._h, dim, _ptr(out, _ip))
        return out

    def neighbors(self, block):
        buf = np.zeros(64, np.int32)
        n = lib().orc_dec_neighbors(self._h, block, _ptr(buf, _ip), 64)
        return buf[:n].tolist()


@dataclass
class OracleSolveResult:
    converged: bool
    constraint_iterations: int
    final_dp: float
    global_l2: float
    global_linf: float
    epochs: np.ndarray
    final_jumps: np.ndarray
    controls: np.ndarray
    global_error: np.ndarray
    blocks_p: list
    block_errors: list


def solve(dec: Decomposition, values, max_outer_iterations=10, tolerance=1e-10, log_errors=False,
          enforce_continuity=True):
    v = np.ascontiguousarray(values, np.float64)
    assert v.shape == dec.grid_dims
    h = C.c_void_p()
    L = lib()
    _check(L.orc_solve(dec._h, _ptr(v, _dp), max_outer_iterations, C.c_double(tolerance), int(log_errors),
                       int(enforce_continuity), C.byref(h)))
    try:
        ints = np.zeros(4, np.int32)
        dbl = np.zeros(3, np.float64)
        L.orc_result_scalars(h, _ptr(ints, _ip), _ptr(dbl, _dp))
        ep = np.zeros((int(ints[2]), 4), np.float64)
        L.orc_result_epochs(h, _ptr(ep, _dp))
        fj = np.zeros((int(ints[3]), 4), np.float64)
        L.orc_result_final_jumps(h, _ptr(fj, _dp))
        ctrl = np.zeros(tuple(int(x) for x in dec.nctrl()), np.float64)
        L.orc_result_controls(h, _ptr(ctrl, _dp))
        err = np.zeros(dec.grid_dims, np.float64)
        L.orc_result_error(h, _ptr(err, _dp))
        bdims = dec.blockdims()
        blocks = []
        for b in range(dec.nblocks):
            shape = tuple(int(bdims[b, d, 9] - bdims[b, d, 8]) for d in range(dec.rank))
            pb = np.zeros(shape, np.float64)
            L.orc_result_block_p(h, b, _ptr(pb, _dp))
            blocks.append(pb)
        berr = []
        if log_errors:
            for e in range(int(ints[2])):
                buf = np.zeros((dec.nblocks, 2), np.float64)
                L.orc_result_block_errors(h, e, _ptr(buf, _dp))
                berr.append(buf)
        return OracleSolveResult(bool(ints[0]), int(ints[1]), float(dbl[0]), float(dbl[1]), float(dbl[2]), ep, fj,
                                 ctrl, err, blocks, berr)
    finally:
        L.orc_result_free(h)
