"""Python host mirror of the reference `mfadd` API for the hot path.

Names, argument meaning and error behaviour follow the reference headers
(/root/reference/proj/core/include/mfadd/{knots,collocation,lsq,decode,layout,
solver}.hpp).  Every numerical result comes from the sm_100a kernels behind
the C ABI (include/mfadd_b200.h); this module only marshals arguments.

Exception mapping (status code -> class, mirroring the reference):
  invalid_argument -> InvalidArgument (a ValueError)
  out_of_range     -> OutOfRange (an IndexError)
  SingularFitError -> SingularFitError(dim, span)
  runtime_error    -> RuntimeFault;  logic_error -> LogicError
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _lib as L

# ------------------------------------------------------------------ errors


class MfaddError(Exception):
    code = -1


class InvalidArgument(MfaddError, ValueError):
    code = L.MFADD_EINVAL


class OutOfRange(MfaddError, IndexError):
    code = L.MFADD_ERANGE


class SingularFitError(MfaddError, RuntimeError):
    """lsq.hpp:24-28: a per-dimension normal matrix is not SPD."""
    code = L.MFADD_ESINGULAR

    def __init__(self, msg, dim=-1, span=-1):
        super().__init__(msg)
        self.dim, self.span = dim, span


class RuntimeFault(MfaddError, RuntimeError):
    code = L.MFADD_ERUNTIME


class LogicError(MfaddError):
    code = L.MFADD_ELOGIC


class CudaError(MfaddError, RuntimeError):
    code = L.MFADD_ECUDA


_BY_CODE = {c.code: c for c in (InvalidArgument, OutOfRange, RuntimeFault, LogicError, CudaError)}


def _check(rc):
    if rc == 0:
        return
    lib = L.load()
    msg = (lib.mfadd_last_error() or b"").decode(errors="replace")
    if rc == L.MFADD_ESINGULAR:
        raise SingularFitError(msg, lib.mfadd_last_error_dim(), lib.mfadd_last_error_span())
    raise _BY_CODE.get(rc, MfaddError)(msg)


def _dp(a):
    return a.ctypes.data_as(L.c_dp)


def _lp(a):
    return a.ctypes.data_as(L.c_lp)


def _ip(a):
    return a.ctypes.data_as(L.c_ip)


# ------------------------------------------------------------------ knots


@dataclass
class KnotVector:
    """knots.hpp:11-30."""
    degree: int
    knots: np.ndarray
    clamp_left: bool = True
    clamp_right: bool = True

    def basis_count(self) -> int:
        return len(self.knots) - self.degree - 1

    def domain_min(self) -> float:
        return float(self.knots[self.degree])

    def domain_max(self) -> float:
        return float(self.knots[self.basis_count()])

    def span_count(self) -> int:
        n = self.basis_count()
        return int(sum(1 for s in range(self.degree, n) if self.knots[s] < self.knots[s + 1]))

    def greville(self, i: int) -> float:
        return float(sum(self.knots[i + j] for j in range(1, self.degree + 1)) / self.degree)


def make_knot_vector(degree, basis_count, a=0.0, b=1.0, clamp_left=True, clamp_right=True) -> KnotVector:
    """knots.cpp:48-81 (host metadata, same floating-point expressions)."""
    if degree < 1:
        raise InvalidArgument("make_knot_vector: degree must be >= 1")
    if basis_count < degree + 1:
        raise InvalidArgument(f"make_knot_vector: basis count must be at least p+1 (got {basis_count} for p={degree})")
    if not a < b:
        raise InvalidArgument("make_knot_vector: range must satisfy a < b")
    p, spans = degree, basis_count - degree
    h = (b - a) / spans
    kn = [a] * (p + 1) if clamp_left else [a - i * h for i in range(p, 0, -1)] + [a]
    kn += [a + k * h for k in range(1, spans)]
    kn += [b] * (p + 1) if clamp_right else [b] + [b + i * h for i in range(1, p + 1)]
    return KnotVector(degree, np.array(kn, np.float64), clamp_left, clamp_right)


# ------------------------------------------------------------------ device context

_default_ctx = None


class Context:
    """One CUDA device + stream (mfadd_context)."""

    def __init__(self, device: int = 0, stream: Optional[int] = None):
        lib = L.load()
        h = C.c_void_p()
        _check(lib.mfadd_context_create(device, C.c_void_p(stream) if stream else None, C.byref(h)))
        self._h = h
        self.device = device

    def launch_count(self) -> int:
        return L.load().mfadd_context_launch_count(self._h)

    def close(self):
        if getattr(self, "_h", None):
            L.load().mfadd_context_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


# ------------------------------------------------------------------ collocation


@dataclass
class BandedCollocation:
    """collocation.hpp:15-49 (host copy of the rows the GPU computed)."""
    rows: int
    cols: int
    band: int
    first_col: np.ndarray
    count: np.ndarray
    values: np.ndarray  # rows x band, clipped values left-aligned

    def row_sum(self, j):
        return float(self.values[j, : self.count[j]].sum())

    def dense(self):
        m = np.zeros((self.rows, self.cols))
        for j in range(self.rows):
            c0 = self.first_col[j]
            m[j, c0:c0 + self.count[j]] = self.values[j, : self.count[j]]
        return m


def collocation_matrix(kv: KnotVector, params, col_lo: int = 0, col_hi: Optional[int] = None,
                       ctx: Optional[Context] = None) -> BandedCollocation:
    """collocation_matrix(kv, params[, col_lo, col_hi]), collocation.hpp:53-58, on the GPU (K1)."""
    ctx = ctx or default_context()
    kn = np.ascontiguousarray(kv.knots, np.float64)
    pm = np.ascontiguousarray(params, np.float64)
    if col_hi is None:
        col_hi = kv.basis_count()
    m = len(pm)
    fc = np.zeros(m, np.int64)
    cnt = np.zeros(m, np.int32)
    vals = np.zeros((m, kv.degree + 1), np.float64)
    if m == 0:
        raise InvalidArgument("collocation_matrix: empty parameter list")
    _check(L.load().mfadd_collocation(ctx._h, _dp(kn), len(kn), kv.degree, _dp(pm), m, col_lo, col_hi, _lp(fc),
                                      _ip(cnt), _dp(vals)))
    return BandedCollocation(m, col_hi - col_lo, kv.degree + 1, fc, cnt, vals)


def find_span(kv: KnotVector, u: float, ctx: Optional[Context] = None) -> int:
    """find_span (knots.hpp:36) on the GPU (mfadd_basis_funs)."""
    return basis_funs_batch(kv, [u], ctx=ctx)[0][0]


@dataclass
class SpanBasis:
    """SpanBasis (knots.hpp:39-50): span, p+1 values, (orders+1) x (p+1) derivative rows (row 0 = values)."""
    span: int
    orders: int
    values: np.ndarray
    derivatives: np.ndarray

    def deriv(self, k, j):
        return float(self.derivatives[k, j])


def basis_funs_batch(kv: KnotVector, us, spans=None, orders: int = 0, ctx: Optional[Context] = None):
    """find_span + basis_funs / basis_derivs for many parameters in one GPU call:
    returns (spans[n], values[n, orders+1, p+1])."""
    ctx = ctx or default_context()
    kn = np.ascontiguousarray(kv.knots, np.float64)
    u = np.ascontiguousarray(us, np.float64).reshape(-1)
    n = len(u)
    out = np.zeros((n, orders + 1, kv.degree + 1), np.float64)
    sp_out = np.zeros(n, np.int32)
    sp_in = None if spans is None else np.ascontiguousarray(spans, np.int32).reshape(-1)
    if sp_in is not None and len(sp_in) != n:
        raise InvalidArgument("basis_funs: spans and parameters differ in length")
    _check(L.load().mfadd_basis_funs(ctx._h, _dp(kn), len(kn), kv.degree, n, _dp(u),
                                     None if sp_in is None else _ip(sp_in), orders, _ip(sp_out), _dp(out)))
    return [int(x) for x in sp_out], out


def basis_funs(kv: KnotVector, span: int, u: float, ctx: Optional[Context] = None) -> SpanBasis:
    """basis_funs (knots.hpp:53): Cox-de Boor values at `span` (a neighbouring
    span gives the one-sided polynomial piece)."""
    sp, v = basis_funs_batch(kv, [u], spans=[span], ctx=ctx)
    return SpanBasis(sp[0], 0, v[0, 0].copy(), v[0].copy())


def basis_derivs(kv: KnotVector, span: int, u: float, k: int, ctx: Optional[Context] = None) -> SpanBasis:
    """basis_derivs (knots.hpp:56): derivative rows 0..k (row 0 = basis_funs)."""
    sp, v = basis_funs_batch(kv, [u], spans=[span], orders=k, ctx=ctx)
    return SpanBasis(sp[0], k, v[0, 0].copy(), v[0].copy())


# ------------------------------------------------------------------ lsq / decode


def _pack(kvs: Sequence[KnotVector], params):
    kn = np.concatenate([np.asarray(k.knots, np.float64) for k in kvs])
    ko = np.cumsum([0] + [len(k.knots) for k in kvs]).astype(np.int64)
    pm = np.concatenate([np.asarray(p, np.float64) for p in params])
    po = np.cumsum([0] + [len(p) for p in params]).astype(np.int64)
    return kn, ko, pm, po


@dataclass
class LocalProblem:
    """lsq.hpp:16-22, described by its ingredients (knot vectors, params,
    column windows) rather than host-built collocation matrices: the GPU
    builds the rows itself."""
    kvs: List[KnotVector]
    params: List[np.ndarray]
    windows: List[tuple]
    q: np.ndarray


def fit_unconstrained(problem: LocalProblem, ctx: Optional[Context] = None) -> np.ndarray:
    """fit_unconstrained (lsq.hpp:33), K1+K2+K3 on the GPU."""
    ctx = ctx or default_context()
    degree = problem.kvs[0].degree
    kn, ko, pm, po = _pack(problem.kvs, problem.params)
    lo = np.array([w[0] for w in problem.windows], np.int64)
    hi = np.array([w[1] for w in problem.windows], np.int64)
    q = np.ascontiguousarray(problem.q, np.float64)
    if q.shape != tuple(len(p) for p in problem.params):
        raise InvalidArgument("LocalProblem: row count mismatch")
    out = np.zeros(tuple(int(h - l) for l, h in zip(lo, hi)), np.float64)
    _check(L.load().mfadd_fit_unconstrained(ctx._h, len(problem.kvs), degree, _dp(kn), _lp(ko), _dp(pm), _lp(po),
                                            _lp(lo), _lp(hi), _dp(q), _dp(out)))
    return out


@dataclass
class ResidualStats:
    """ResidualStats (lsq.hpp:35-39)."""
    l2: float
    linf: float
    pointwise: Optional[np.ndarray]


def residual_error(problem: LocalProblem, controls, want_pointwise: bool = True,
                   ctx: Optional[Context] = None) -> ResidualStats:
    """residual_error (lsq.hpp:41, lsq.cpp:66-85) on the GPU: decode of the
    window-clipped rows, pointwise q - decode bitwise equal to the reference."""
    ctx = ctx or default_context()
    degree = problem.kvs[0].degree
    kn, ko, pm, po = _pack(problem.kvs, problem.params)
    lo = np.array([w[0] for w in problem.windows], np.int64)
    hi = np.array([w[1] for w in problem.windows], np.int64)
    q = np.ascontiguousarray(problem.q, np.float64)
    if q.shape != tuple(len(p) for p in problem.params):
        raise InvalidArgument("LocalProblem: row count mismatch")
    c = np.ascontiguousarray(controls, np.float64)
    if c.shape != tuple(int(h - l) for l, h in zip(lo, hi)):
        raise InvalidArgument("residual_error: control extents do not match the column windows")
    pw = np.zeros(q.shape, np.float64) if want_pointwise else None
    l2 = C.c_double()
    li = C.c_double()
    _check(L.load().mfadd_residual_error(ctx._h, len(problem.kvs), degree, _dp(kn), _lp(ko), _dp(pm), _lp(po),
                                         _lp(lo), _lp(hi), _dp(q), _dp(c), None if pw is None else _dp(pw),
                                         C.byref(l2), C.byref(li)))
    return ResidualStats(l2.value, li.value, pw)


def decode(controls, kvs: Sequence[KnotVector], params, col_offset=None, ctx: Optional[Context] = None):
    """decode (decode.hpp:20-22), K1 + K7 on the GPU."""
    ctx = ctx or default_context()
    c = np.ascontiguousarray(controls, np.float64)
    if c.ndim != len(kvs) or len(kvs) != len(params):
        raise InvalidArgument("decode: dimension mismatch between lattice, knot vectors and parameters")
    kn, ko, pm, po = _pack(kvs, params)
    ext = np.array(c.shape, np.int64)
    off = None if col_offset is None or len(col_offset) == 0 else np.array(col_offset, np.int64)
    out = np.zeros(tuple(len(p) for p in params), np.float64)
    _check(L.load().mfadd_decode(ctx._h, len(kvs), kvs[0].degree, _dp(kn), _lp(ko), _dp(pm), _lp(po), _lp(ext),
                                 None if off is None else _lp(off), _dp(c), _dp(out)))
    return out


# ------------------------------------------------------------------ layout

BLOCKDIM_FIELDS = ("span_lo", "span_hi", "delta_lo", "delta_hi", "overlap_lo", "overlap_hi", "local_span_lo",
                   "local_span_hi", "dof_lo", "dof_hi", "own_lo", "own_hi", "input_lo", "input_hi",
                   "own_input_lo", "own_input_hi")


@dataclass
class BlockDim:
    """layout.hpp:47-57."""
    span_lo: int
    span_hi: int
    delta_lo: int
    delta_hi: int
    overlap_lo: int
    overlap_hi: int
    local_span_lo: int
    local_span_hi: int
    dof_lo: int
    dof_hi: int
    own_lo: int
    own_hi: int
    input_lo: int
    input_hi: int
    own_input_lo: int
    own_input_hi: int


@dataclass
class BlockLayout:
    """layout.hpp:59-66."""
    id: int
    coords: List[int]
    dims: List[BlockDim]
    neighbors: List[int]

    def holds(self, dof):
        return all(d.dof_lo <= i < d.dof_hi for d, i in zip(self.dims, dof))

    def owns(self, dof):
        return all(d.own_lo <= i < d.own_hi for d, i in zip(self.dims, dof))


def delta_width(degree: int) -> int:
    """layout.cpp:11-14."""
    if degree < 1:
        raise InvalidArgument("delta_width: degree must be >= 1")
    return degree // 2


class SharedDofMap:
    """layout.hpp:70-92 (host view of the partition's holder ranges)."""

    def __init__(self, dec: "Decomposition"):
        self._dec = dec
        self._hr = [dec._holder_ranges(k) for k in range(dec.rank)]

    def holder_span(self, dim, i):
        r = self._hr[dim][i]
        return int(r[0]), int(r[1])

    def n_s(self, dof):
        c = 1
        for k, i in enumerate(dof):
            r = self._hr[k][i]
            c *= int(r[1] - r[0] + 1)
        return c

    def classify(self, dof):
        c = self.n_s(dof)
        return "interior" if c <= 1 else ("singly_shared" if c == 2 else "multi_shared")

    def weight(self, dof):
        return 1.0 / self.n_s(dof)

    def holders(self, dof):
        import itertools
        ranges = [range(int(self._hr[k][i][0]), int(self._hr[k][i][1]) + 1) for k, i in enumerate(dof)]
        ids = []
        for c in itertools.product(*ranges):
            bid = 0
            for k, ck in enumerate(c):
                bid = bid * self._dec.blocks_per_dim[k] + ck
            ids.append(bid)
        return sorted(ids)

    def any_shared(self):
        return bool(L.load().mfadd_dec_any_shared(self._dec._h))

    def for_each_shared(self, fn):
        import itertools
        for dof in itertools.product(*[range(int(n)) for n in self._dec.n_ctrl]):
            c = self.n_s(dof)
            if c > 1:
                fn(dof, c)


class Decomposition:
    """layout.hpp:94-104 (`partition()` result), held by the C ABI."""

    def __init__(self, handle, grid_dims, bounds, blocks_per_dim, degree, overlap, clamp):
        self._h = handle
        lib = L.load()
        self.rank = lib.mfadd_dec_rank(handle)
        self.nblocks = lib.mfadd_dec_block_count(handle)
        self.grid_dims = tuple(int(x) for x in grid_dims)
        self.bounds = [tuple(b) for b in bounds]
        self.blocks_per_dim = [int(b) for b in blocks_per_dim]
        self.degree = degree
        self.overlap = 0 if clamp else int(overlap)
        self.clamp_interfaces = bool(clamp)
        nc = np.zeros(self.rank, np.int64)
        lib.mfadd_dec_nctrl(handle, _lp(nc))
        self.n_ctrl = [int(x) for x in nc]
        self.kvs = []
        for k in range(self.rank):
            n = lib.mfadd_dec_knots(handle, k, None)
            kn = np.zeros(n, np.float64)
            lib.mfadd_dec_knots(handle, k, _dp(kn))
            self.kvs.append(KnotVector(degree, kn, True, True))
        bd = self.block_dims_array()
        co = np.zeros((self.nblocks, self.rank), np.int32)
        lib.mfadd_dec_coords(handle, _ip(co))
        buf = np.zeros(64, np.int32)
        self.blocks = []
        for b in range(self.nblocks):
            nn = lib.mfadd_dec_neighbors(handle, b, _ip(buf), 64)
            self.blocks.append(BlockLayout(b, co[b].tolist(), [BlockDim(*map(int, bd[b, k])) for k in range(self.rank)],
                                           buf[:nn].tolist()))
        self.shared = SharedDofMap(self)

    def __del__(self):
        if getattr(self, "_h", None):
            try:
                L.load().mfadd_decomposition_free(self._h)
            except Exception:
                pass
            self._h = None

    def block_dims_array(self):
        out = np.zeros((self.nblocks, self.rank, 16), np.int64)
        L.load().mfadd_dec_block_dims(self._h, _lp(out))
        return out

    def _holder_ranges(self, dim):
        out = np.zeros((self.n_ctrl[dim], 2), np.int32)
        L.load().mfadd_dec_holder_ranges(self._h, dim, _ip(out))
        return out

    def shared_dof_box(self, a, b):
        box = []
        for da, db in zip(self.blocks[a].dims, self.blocks[b].dims):
            lo, hi = max(da.dof_lo, db.dof_lo), min(da.dof_hi, db.dof_hi)
            if lo >= hi:
                return []
            box.append((lo, hi))
        return box

    def exchange_volume(self):
        out = np.zeros(self.nblocks, np.int64)
        L.load().mfadd_dec_exchange_volume(self._h, _lp(out))
        return out

    def compression_ratio(self):
        return L.load().mfadd_dec_compression_ratio(self._h)

    def span_count(self, dim):
        return self.kvs[dim].span_count()

    def total_inputs(self):
        return int(np.prod(self.grid_dims))


def partition(grid_dims, bounds, blocks_per_dim, degree, nctrl_per_block, overlap, clamp_interfaces=False):
    """partition (layout.hpp:107-111)."""
    rank = len(grid_dims)
    if not (len(bounds) == len(blocks_per_dim) == len(nctrl_per_block) == rank):
        raise InvalidArgument("partition: per-dimension argument counts disagree")
    g = np.array(grid_dims, np.int64)
    bd = np.array(bounds, np.float64).reshape(-1)
    bp = np.array(blocks_per_dim, np.int32)
    nc = np.array(nctrl_per_block, np.int64)
    h = C.c_void_p()
    _check(L.load().mfadd_partition(rank, _lp(g), _dp(bd), _ip(bp), degree, _lp(nc), overlap, int(clamp_interfaces),
                                    C.byref(h)))
    return Decomposition(h, grid_dims, bounds, blocks_per_dim, degree, overlap, clamp_interfaces)


def compression_ratio(dec: Decomposition) -> float:
    return dec.compression_ratio()


def exchange_volume(dec: Decomposition):
    return dec.exchange_volume()


# ------------------------------------------------------------------ solver


@dataclass
class Field:
    """field.hpp:17-29: row-major samples, last dim fastest, u_j = j/(m-1)."""
    dims: List[int]
    bounds: List[tuple]
    values: np.ndarray
    name: str = ""

    def rank(self):
        return len(self.dims)

    def coordinate(self, dim, j):
        a, b = self.bounds[dim]
        m = self.dims[dim]
        return a if m == 1 else a + (b - a) * float(j) / float(m - 1)

    def parameter_grid(self, dim):
        m = self.dims[dim]
        return np.array([0.0 if m == 1 else float(j) / float(m - 1) for j in range(m)])

    def validate(self):
        if not self.dims or len(self.dims) != len(self.bounds):
            raise InvalidArgument("Field: dims/bounds mismatch")
        for d, (a, b) in zip(self.dims, self.bounds):
            if d < 2:
                raise InvalidArgument("Field: need at least 2 points per dimension")
            if not a < b:
                raise InvalidArgument("Field: bounds min must be < max")
        if int(np.prod(self.dims)) != int(np.asarray(self.values).size):
            raise InvalidArgument("Field: value count does not match extents")


@dataclass
class SolverConfig:
    """solver.hpp:16-22 (+ store_error: materialise global_error)."""
    max_outer_iterations: int = 10
    tolerance: float = 1e-10
    workers: int = 1
    log_errors: bool = True
    enforce_continuity: bool = True
    store_error: bool = True

    def to_c(self):
        return L.SolverConfigC(self.max_outer_iterations, self.tolerance, self.workers, int(self.log_errors),
                               int(self.enforce_continuity), int(self.store_error))


@dataclass
class InterfaceJump:
    block_a: int
    block_b: int
    linf_ss: float
    linf_ms: float


@dataclass
class EpochStats:
    iteration: int
    dp_max: float
    jump_ss: float
    jump_ms: float
    block_errors: list = field(default_factory=list)


@dataclass
class PhaseTimings:
    setup: float = 0.0
    local_solve: float = 0.0
    exchange: float = 0.0
    constraint: float = 0.0
    decode: float = 0.0


@dataclass
class MfaModel:
    """model.hpp:18-35: global knot vectors, the converged control lattice,
    domain bounds and run provenance.  eval / eval_deriv / decode_grid run on
    the GPU (model.cu)."""
    degrees: List[int]
    kvs: List[KnotVector]
    controls: np.ndarray
    bounds: List[tuple]
    provenance: dict = field(default_factory=dict)

    def rank(self) -> int:
        return len(self.kvs)

    def validate(self):
        """model.cpp:11-24."""
        if not self.kvs or len(self.kvs) != len(self.degrees) or len(self.kvs) != len(self.bounds):
            raise InvalidArgument("MfaModel: inconsistent dimension counts")
        if np.asarray(self.controls).ndim != self.rank():
            raise InvalidArgument("MfaModel: control lattice rank mismatch")
        for d, kv in enumerate(self.kvs):
            if kv.degree != self.degrees[d]:
                raise InvalidArgument(f"MfaModel: degree mismatch in dimension {d}")
            if kv.basis_count() != np.asarray(self.controls).shape[d]:
                raise InvalidArgument(f"MfaModel: control extent must equal #knots - p - 1 in dimension {d}")

    def param_of(self, dim, x) -> float:
        """model.cpp:26-29."""
        a, b = self.bounds[dim]
        return (x - a) / (b - a)

    def eval(self, params, ctx: Optional[Context] = None) -> float:
        """model.cpp:31-33."""
        return float(eval_points(self.controls, self.kvs, np.asarray(params, np.float64)[None, :], ctx=ctx)[0])

    def eval_deriv(self, params, orders, ctx: Optional[Context] = None) -> float:
        """model.cpp:35-37."""
        return float(eval_points(self.controls, self.kvs, np.asarray(params, np.float64)[None, :], orders,
                                 ctx=ctx)[0])

    def decode_grid(self, res, ctx: Optional[Context] = None) -> np.ndarray:
        """model.cpp:39-49 (GPU decode at u_j = j / (res - 1))."""
        ctx = ctx or default_context()
        if len(res) != self.rank():
            raise InvalidArgument("decode_grid: resolution rank mismatch")
        if len(set(self.degrees)) != 1:
            raise InvalidArgument("decode_grid: mixed per-dimension degrees are not supported")
        c = np.ascontiguousarray(self.controls, np.float64)
        kn, ko = _pack_knots(self.kvs)
        r = np.array(res, np.int64)
        out = np.zeros(tuple(int(x) for x in res) if all(x >= 2 for x in res) else (1,), np.float64)
        _check(L.load().mfadd_decode_grid(ctx._h, self.rank(), self.degrees[0], _dp(kn), _lp(ko),
                                          _lp(np.array(c.shape, np.int64)), _dp(c), _lp(r), _dp(out)))
        return out


class Side:
    """decode.hpp:24."""
    Below = 0
    Above = 1


def _pack_knots(kvs):
    kn = np.ascontiguousarray(np.concatenate([np.asarray(k.knots, np.float64) for k in kvs]))
    ko = np.zeros(len(kvs) + 1, np.int64)
    for i, k in enumerate(kvs):
        ko[i + 1] = ko[i] + len(k.knots)
    return kn, ko


def eval_points(controls, kvs: Sequence[KnotVector], points, orders=None, side_dim: int = -1, side: int = Side.Above,
                col_offset=None, ctx: Optional[Context] = None) -> np.ndarray:
    """Batched eval_deriv / eval_deriv_sided (decode.hpp:28-40) on the GPU:
    points [npts][rank] -> values [npts], bitwise equal to the reference."""
    ctx = ctx or default_context()
    c = np.ascontiguousarray(controls, np.float64)
    pts = np.ascontiguousarray(np.atleast_2d(np.asarray(points, np.float64)))
    if c.ndim != len(kvs) or pts.shape[1] != len(kvs):
        raise InvalidArgument("decode: dimension mismatch between lattice, knot vectors and parameters")
    kn, ko = _pack_knots(kvs)
    deg = np.array([k.degree for k in kvs], np.int32)
    ords = None if orders is None or len(orders) == 0 else np.array(orders, np.int32)
    off = None if col_offset is None or len(col_offset) == 0 else np.array(col_offset, np.int64)
    out = np.zeros(pts.shape[0], np.float64)
    _check(L.load().mfadd_eval_points(ctx._h, len(kvs), _ip(deg), _dp(kn), _lp(ko), _lp(np.array(c.shape, np.int64)),
                                      None if off is None else _lp(off), _dp(c), pts.shape[0], _dp(pts),
                                      None if ords is None else _ip(ords), side_dim, side, _dp(out)))
    return out


def eval_deriv(controls, kvs, point, orders=None, col_offset=None, ctx: Optional[Context] = None) -> float:
    """decode.hpp:28-30."""
    return float(eval_points(controls, kvs, np.asarray(point, np.float64)[None, :], orders, -1, Side.Above,
                             col_offset, ctx)[0])


def eval_deriv_sided(controls, kvs, point, orders, side_dim, side, col_offset=None,
                     ctx: Optional[Context] = None) -> float:
    """decode.hpp:35-38."""
    return float(eval_points(controls, kvs, np.asarray(point, np.float64)[None, :], orders, side_dim, side,
                             col_offset, ctx)[0])


def continuity_jumps(model: MfaModel, dim: int, u_interface: float, max_order: int, cross_samples: int = 5,
                     ctx: Optional[Context] = None) -> List[float]:
    """solver.hpp:96 (assembled-model variant); probe points evaluated on the GPU."""
    ctx = ctx or default_context()
    c = np.ascontiguousarray(model.controls, np.float64)
    kn, ko = _pack_knots(model.kvs)
    deg = np.array(model.degrees, np.int32)
    out = np.zeros(max(max_order, 0) + 1, np.float64)
    _check(L.load().mfadd_continuity_jumps(ctx._h, model.rank(), _ip(deg), _dp(kn), _lp(ko),
                                           _lp(np.array(c.shape, np.int64)), _dp(c), dim, float(u_interface),
                                           max_order, cross_samples, _dp(out)))
    return [float(x) for x in out]


def write_mfa(model: MfaModel, path) -> None:
    """model.hpp:40: MFDD v1 container, bit-exact with the reference writer."""
    c = np.ascontiguousarray(model.controls, np.float64)
    kn, ko = _pack_knots(model.kvs)
    deg = np.array(model.degrees, np.int32)
    cl = np.array([1 if k.clamp_left else 0 for k in model.kvs], np.uint8)
    cr = np.array([1 if k.clamp_right else 0 for k in model.kvs], np.uint8)
    bnd = np.ascontiguousarray(np.array(model.bounds, np.float64).reshape(-1))
    keys = [str(k).encode() for k in model.provenance]
    vals = [str(model.provenance[k]).encode() for k in model.provenance]
    v = L.ModelViewC()
    v.rank = len(model.kvs)
    v.degrees = _ip(deg)
    v.clamp_left = cl.ctypes.data_as(C.POINTER(C.c_ubyte))
    v.clamp_right = cr.ctypes.data_as(C.POINTER(C.c_ubyte))
    v.knots = _dp(kn)
    v.kn_off = _lp(ko)
    ext = np.array(c.shape, np.int64)
    v.ctrl_ext = _lp(ext)
    v.bounds = _dp(bnd)
    v.nprov = len(keys)
    karr = (C.c_char_p * max(len(keys), 1))(*keys)
    varr = (C.c_char_p * max(len(vals), 1))(*vals)
    v.prov_keys = C.cast(karr, C.POINTER(C.c_char_p))
    v.prov_values = C.cast(varr, C.POINTER(C.c_char_p))
    v.controls = _dp(c)
    _check(L.load().mfadd_write_mfa(str(path).encode(), C.byref(v)))


def read_mfa(path) -> MfaModel:
    """model.hpp:41."""
    lib = L.load()
    h = C.c_void_p()
    _check(lib.mfadd_read_mfa(str(path).encode(), C.byref(h)))
    try:
        v = L.ModelViewC()
        _check(lib.mfadd_model_view_of(h, C.byref(v)))
        r = v.rank
        ko = [int(v.kn_off[i]) for i in range(r + 1)]
        ext = [int(v.ctrl_ext[i]) for i in range(r)]
        kvs = []
        for d in range(r):
            kn = np.array([v.knots[i] for i in range(ko[d], ko[d + 1])], np.float64)
            kvs.append(KnotVector(int(v.degrees[d]), kn, bool(v.clamp_left[d]), bool(v.clamp_right[d])))
        n = int(np.prod(ext))
        ctrl = np.ctypeslib.as_array(v.controls, shape=(n,)).copy().reshape(ext)
        bounds = [(float(v.bounds[2 * d]), float(v.bounds[2 * d + 1])) for d in range(r)]
        prov = {v.prov_keys[i].decode(): v.prov_values[i].decode() for i in range(v.nprov)}
        return MfaModel([int(v.degrees[d]) for d in range(r)], kvs, ctrl, bounds, prov)
    finally:
        lib.mfadd_model_free(h)


class RawScalar:
    """field.hpp:43."""
    Float32 = 0
    Float64 = 1


class RawByteOrder:
    """field.hpp:44."""
    Little = 0
    Big = 1


def read_raw_grid(path, dims, type: int, order: int = RawByteOrder.Little, bounds=None, device_out=None,
                  ctx: Optional[Context] = None):
    """field.hpp:48-50: the bytes are copied to the device and byte-swapped /
    widened to fp64 there (model.cu k_raw_to_f64).  With `device_out` (a CUDA
    pointer of prod(dims) doubles, e.g. torch tensor.data_ptr()) the field
    stays in HBM and only the Field metadata is returned."""
    ctx = ctx or default_context()
    import os
    dims = [int(d) for d in dims]
    d_arr = np.array(dims, np.int64)
    values = None
    if device_out is None:
        values = np.zeros(int(np.prod(dims)) if dims else 0, np.float64)
        ptr, on_dev = values.ctypes.data_as(C.c_void_p), 0
    else:
        ptr, on_dev = C.c_void_p(int(device_out)), 1
    _check(L.load().mfadd_read_raw_grid(ctx._h, str(path).encode(), len(dims), _lp(d_arr), int(type), int(order), ptr,
                                        on_dev))
    b = list(bounds) if bounds else [(0.0, 1.0)] * len(dims)
    if len(b) != len(dims):
        raise InvalidArgument("read_raw_grid: bounds/dims mismatch")
    return Field(dims, b, None if values is None else values.reshape(dims), os.path.basename(str(path)))


@dataclass
class BlockState:
    id: int
    col_offset: List[int]
    p: np.ndarray


@dataclass
class SolveResult:
    model: MfaModel
    converged: bool
    constraint_iterations: int
    final_dp: float
    epochs: List[EpochStats]
    final_jumps: List[InterfaceJump]
    timings: PhaseTimings
    blocks: List[BlockState]
    global_l2: float
    global_linf: float
    global_error: Optional[np.ndarray]


class Comm:
    """An NCCL communicator for sharded solves (one rank per GPU process)."""

    def __init__(self, unique_id: bytes, rank: int, nranks: int, ctx: Optional["Context"] = None):
        self.ctx = ctx or default_context()
        self.rank, self.nranks = rank, nranks
        buf = C.create_string_buffer(bytes(unique_id), 128)
        h = C.c_void_p()
        _check(L.load().mfadd_comm_create(self.ctx._h, buf, rank, nranks, C.byref(h)))
        self._h = h

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(L.load().mfadd_nccl_unique_id(buf))
        return buf.raw

    def close(self):
        if getattr(self, "_h", None):
            L.load().mfadd_comm_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def shard_range(dec: "Decomposition", rank: int, nranks: int):
    """(block_lo, block_hi, input_row_lo, input_row_hi) of `rank` (host-side plan)."""
    blo, bhi, ilo, ihi = C.c_int(), C.c_int(), C.c_int64(), C.c_int64()
    _check(L.load().mfadd_shard_range(dec._h, rank, nranks, C.byref(blo), C.byref(bhi), C.byref(ilo), C.byref(ihi)))
    return blo.value, bhi.value, ilo.value, ihi.value


def shard_box(dec: "Decomposition", rank: int, nranks: int):
    """(box_lo, box_hi): the axis-0 input rows `rank`'s sharded solve reads (its slab)."""
    lo, hi = C.c_int64(), C.c_int64()
    _check(L.load().mfadd_shard_box(dec._h, rank, nranks, C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


def shard_ctrl_rows(dec: "Decomposition", rank: int, nranks: int):
    """(own_lo, own_hi): the lattice rows along axis 0 `rank` owns."""
    lo, hi = C.c_int64(), C.c_int64()
    _check(L.load().mfadd_shard_ctrl_rows(dec._h, rank, nranks, C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


def shard_exchange(dec: "Decomposition", rank: int, nranks: int, peer: int, recv: bool) -> np.ndarray:
    """Per-epoch exchange layout of `rank` with `peer`: rows (holder block, i0, i1, i2) in buffer order."""
    lib = L.load()
    n = lib.mfadd_shard_exchange(dec._h, rank, nranks, peer, int(recv), None, 0)
    if n < 0:
        _check(-n)
    out = np.zeros((n, 4), np.int64)
    if n:
        lib.mfadd_shard_exchange(dec._h, rank, nranks, peer, int(recv), out.ctypes.data_as(C.POINTER(C.c_int64)), n)
    return out


def solve_loopback(field_: "Field", dec: "Decomposition", nranks: int, config: "SolverConfig" = None,
                   ctx: Optional["Context"] = None) -> "SolveResult":
    """The sharded solve with all `nranks` shard solvers in this process on one
    device (device-to-device copies stand in for NCCL): checks the multi-GPU
    path against the single-device solve."""
    ctx = ctx or default_context()
    config = config or SolverConfig()
    cfg = config.to_c()
    v = np.ascontiguousarray(field_.values, np.float64).reshape(-1)
    ctrl = np.zeros(tuple(dec.n_ctrl), np.float64)
    err = np.zeros(dec.grid_dims, np.float64)
    sm = L.SolveSummaryC()
    ep = (L.EpochStatsC * (config.max_outer_iterations + 2))()
    npairs = sum(len([j for j in b.neighbors if j > b.id]) for b in dec.blocks)
    fj = np.zeros((max(1, npairs), 4))
    _check(L.load().mfadd_solve_loopback(ctx._h, dec._h, C.byref(cfg), nranks, v.ctypes.data_as(C.c_void_p),
                                         ctrl.ctypes.data_as(C.c_void_p), err.ctypes.data_as(C.c_void_p),
                                         C.byref(sm), ep, len(ep), _dp(fj), len(fj)))
    epochs = [EpochStats(e.iteration, e.dp_max, e.jump_ss, e.jump_ms) for e in ep[:sm.n_epochs]]
    jumps = [InterfaceJump(int(r[0]), int(r[1]), float(r[2]), float(r[3])) for r in fj[:sm.n_final_jumps]]
    model = MfaModel([dec.degree] * dec.rank, dec.kvs, ctrl, dec.bounds)
    t = PhaseTimings(sm.t_setup, sm.t_local_solve, sm.t_exchange, sm.t_constraint, sm.t_decode)
    return SolveResult(model, bool(sm.converged), sm.constraint_iterations, sm.final_dp, epochs, jumps, t, [],
                       sm.global_l2, sm.global_linf, err)


class Solver:
    """A solve() plan: the decomposition's device tables + work buffers.  With
    `comm`, the plan of this rank's shard (mfadd_solver_create_sharded); run()
    is then collective over the communicator's ranks."""

    def __init__(self, dec: Decomposition, config: SolverConfig = None, ctx: Optional[Context] = None,
                 comm: Optional[Comm] = None):
        self.ctx = ctx or default_context()
        self.dec = dec
        self.config = config or SolverConfig()
        self.comm = comm
        self._cfg = self.config.to_c()
        h = C.c_void_p()
        if comm is None:
            _check(L.load().mfadd_solver_create(self.ctx._h, dec._h, C.byref(self._cfg), C.byref(h)))
        else:
            _check(L.load().mfadd_solver_create_sharded(self.ctx._h, dec._h, C.byref(self._cfg), comm._h,
                                                        C.byref(h)))
        self._h = h
        self.summary = L.SolveSummaryC()
        self._n_field = None   # dec.total_inputs(), read once
        self._buf_seen = None  # (id, side, size) of the last tensor that passed _buf, and its address

    def close(self):
        if getattr(self, "_h", None):
            L.load().mfadd_solver_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # Buffer checks before any pointer crosses the C ABI (the ABI takes plain
    # pointers and sizes; the reference throws invalid_argument for a field
    # whose extents disagree with the decomposition, solver.cpp:335-338).
    def _buf(self, a, n, what, device, shape=None):
        """Address of a float64, C-contiguous buffer of n elements on the right side
        (a multi-dimensional buffer must also have `shape`, e.g. the grid extents)."""
        # a stream of solves on one tensor: the checks ran on its first solve
        # (the host gap between solves counts against every solve's time)
        seen = getattr(self, "_buf_seen", None)
        if seen is not None and seen[0] is a and seen[1] == (device, n) and not isinstance(a, np.ndarray):
            if a.data_ptr() == seen[2] and a.numel() == n:
                return seen[2]
        sh = getattr(a, "shape", None)
        if shape is not None and sh is not None and len(sh) > 1 and tuple(int(x) for x in sh) != tuple(shape):
            raise InvalidArgument("solve: field extents disagree with the decomposition")
        if isinstance(a, np.ndarray):
            if device:
                raise InvalidArgument(f"{what}: expected a device buffer, got a host numpy array")
            if a.dtype != np.float64 or not a.flags["C_CONTIGUOUS"]:
                raise InvalidArgument(f"{what}: expected a C-contiguous float64 array")
            if a.size != n:
                raise InvalidArgument(f"{what}: {a.size} elements, expected {n}")
            return a.ctypes.data
        dt = getattr(a, "dtype", None)
        if dt is not None and str(dt) not in ("torch.float64", "float64"):
            raise InvalidArgument(f"{what}: expected float64, got {dt}")
        if hasattr(a, "is_contiguous") and not a.is_contiguous():
            raise InvalidArgument(f"{what}: expected a contiguous tensor")
        numel = a.numel() if hasattr(a, "numel") else None
        if numel is not None and numel != n:
            raise InvalidArgument(f"{what}: {numel} elements, expected {n}")
        is_cuda = getattr(a, "is_cuda", None)
        if is_cuda is not None and bool(is_cuda) != bool(device):
            raise InvalidArgument(f"{what}: expected a {'device' if device else 'host'} buffer")
        if device and is_cuda and getattr(a, "device", None) is not None and a.device.index not in (None, self.ctx.device):
            raise InvalidArgument(f"{what}: tensor on cuda:{a.device.index}, solver on cuda:{self.ctx.device}")
        ptr = a.data_ptr()
        if shape is not None and hasattr(a, "is_contiguous"):  # (fields only: outputs differ per call)
            self._buf_seen = (a, (device, n), ptr)
        return ptr

    def _field_n(self):
        if getattr(self, "_n_field", None) is None:
            self._n_field = self.dec.total_inputs()
        return self._n_field

    def _ctrl_n(self):
        return int(np.prod(self.dec.n_ctrl))

    # field: numpy array (host) or a torch tensor (host or, with on_device, device)
    def run(self, values, on_device: bool = False):
        lib = L.load()
        if on_device:
            ptr = self._buf(values, self._field_n(), "solve: field", True, self.dec.grid_dims)
            _check(lib.mfadd_solve(self._h, C.c_void_p(ptr), 1, C.byref(self.summary)))
        else:
            v = np.ascontiguousarray(values, np.float64)
            if v.size != self.dec.total_inputs() or (v.ndim > 1 and v.shape != tuple(self.dec.grid_dims)):
                raise InvalidArgument("solve: field extents disagree with the decomposition")
            _check(lib.mfadd_solve(self._h, v.ctypes.data_as(C.c_void_p), 0, C.byref(self.summary)))
        return self.summary

    def run_host(self, values, out_controls, out_error=None):
        """mfadd_solve_host: H2D + solve + D2H in one call (the e2e path)."""
        fp = self._buf(values, self._field_n(), "solve: field", False, self.dec.grid_dims)
        cp = self._buf(out_controls, self._ctrl_n(), "solve: out_controls", False)
        ep = None if out_error is None else C.c_void_p(self._buf(out_error, self._field_n(), "solve: out_error", False))
        _check(L.load().mfadd_solve_host(self._h, C.c_void_p(fp), C.c_void_p(cp), ep, C.byref(self.summary)))
        return self.summary

    def run_host_batch(self, fields, out_controls, out_errors=None):
        """mfadd_solve_host_batch: a stream of solves on host buffers with the
        copies of neighbouring steps overlapped.  Returns the n summaries."""
        n = len(fields)
        if len(out_controls) != n or (out_errors is not None and len(out_errors) != n):
            raise InvalidArgument("solve_host_batch: fields and outputs differ in length")
        fp = (C.c_void_p * n)(*[self._buf(f, self._field_n(), "solve: field", False, self.dec.grid_dims) for f in fields])
        cp = (C.c_void_p * n)(*[self._buf(o, self._ctrl_n(), "solve: out_controls", False) for o in out_controls])
        ep = None if out_errors is None else \
            (C.c_void_p * n)(*[self._buf(o, self._field_n(), "solve: out_error", False) for o in out_errors])
        sums = (L.SolveSummaryC * n)()
        _check(L.load().mfadd_solve_host_batch(self._h, n, fp, cp, ep, sums))
        self.summary = sums[n - 1]
        return list(sums)

    def gather_controls(self):
        """Collective (sharded solver): every rank's owned lattice rows to every rank."""
        _check(L.load().mfadd_solver_gather_controls(self._h))

    def set_profiling(self, on: bool = True):
        _check(L.load().mfadd_solver_set_profiling(self._h, int(on)))

    def kernel_times(self):
        """[(name, ms)] per kernel launch of the last solve (CUDA events on the launching stream)."""
        cap, nl = 4096, 32
        names = C.create_string_buffer(cap * nl)
        ms = np.zeros(cap)
        n = L.load().mfadd_solver_kernel_times(self._h, names, nl, _dp(ms), cap)
        raw = names.raw
        return [(raw[i * nl:(i + 1) * nl].split(b"\0")[0].decode(), float(ms[i])) for i in range(min(n, cap))]

    def continuity_probe(self, probe_order: int = -1, cross_samples: int = 5):
        """The pipeline's continuity probe (pipeline.cpp:210-228) over every
        interior interface of the last solve, on the device-resident block
        lattices: returns (order, jumps[0..order])."""
        out = np.zeros(max(probe_order, self.dec.degree - 1, 0) + 1, np.float64)
        o = C.c_int()
        _check(L.load().mfadd_solver_continuity_probe(self._h, probe_order, cross_samples, _dp(out), C.byref(o)))
        return o.value, [float(x) for x in out[:o.value + 1]]

    def last_launches(self) -> int:
        return L.load().mfadd_solver_last_launches(self._h)

    def device_controls_ptr(self) -> int:
        return L.load().mfadd_solver_device_controls(self._h)

    def result(self, want_blocks: bool = True, want_error: bool = True) -> SolveResult:
        lib = L.load()
        s = self.summary
        ep = (L.EpochStatsC * max(1, s.n_epochs))()
        n = lib.mfadd_solver_epochs(self._h, ep, len(ep))
        epochs = [EpochStats(e.iteration, e.dp_max, e.jump_ss, e.jump_ms) for e in ep[:n]]
        if self.config.log_errors:
            buf = np.zeros((self.dec.nblocks, 2))
            for i, e in enumerate(epochs):
                _check(lib.mfadd_solver_block_errors(self._h, i, _dp(buf)))
                e.block_errors = [tuple(r) for r in buf]
        fj = np.zeros((max(1, s.n_final_jumps), 4))
        nj = lib.mfadd_solver_final_jumps(self._h, _dp(fj), len(fj))
        jumps = [InterfaceJump(int(r[0]), int(r[1]), float(r[2]), float(r[3])) for r in fj[:nj]]
        ctrl = np.zeros(tuple(self.dec.n_ctrl), np.float64)
        _check(lib.mfadd_solver_controls(self._h, ctrl.ctypes.data_as(C.c_void_p), 0))
        err = None
        if want_error and self.config.store_error:
            err = np.zeros(self.dec.grid_dims, np.float64)
            _check(lib.mfadd_solver_global_error(self._h, err.ctypes.data_as(C.c_void_p), 0))
        blocks = []
        if want_blocks:
            for b in self.dec.blocks:
                shape = tuple(d.dof_hi - d.dof_lo for d in b.dims)
                pb = np.zeros(shape, np.float64)
                _check(lib.mfadd_solver_block_controls(self._h, b.id, pb.ctypes.data_as(C.c_void_p), 0))
                blocks.append(BlockState(b.id, [d.dof_lo for d in b.dims], pb))
        model = MfaModel([self.dec.degree] * self.dec.rank, self.dec.kvs, ctrl, self.dec.bounds)
        t = PhaseTimings(s.t_setup, s.t_local_solve, s.t_exchange, s.t_constraint, s.t_decode)
        return SolveResult(model, bool(s.converged), s.constraint_iterations, s.final_dp, epochs, jumps, t, blocks,
                           s.global_l2, s.global_linf, err)


def solve(field_: Field, dec: Decomposition, config: SolverConfig = None, ctx: Optional[Context] = None) -> SolveResult:
    """solve (solver.hpp:76) on the GPU."""
    config = config or SolverConfig()
    if config.max_outer_iterations < 1:
        raise InvalidArgument("SolverConfig: max iterations must be >= 1")
    if not config.tolerance > 0.0:
        raise InvalidArgument("SolverConfig: tolerance must be > 0")
    field_.validate()
    if list(field_.dims) != list(dec.grid_dims):
        raise InvalidArgument("solve: field extents disagree with the decomposition")
    s = Solver(dec, config, ctx)
    try:
        s.run(np.ascontiguousarray(field_.values, np.float64).reshape(-1))
        return s.result()
    finally:
        s.close()
