"""B200-native domain-decomposed MFA encode (arXiv 2210.06528 hot path).

Drop-in for the reference `mfadd` core API on the encode path: partition ->
solve -> (model, error).  All numerics run in sm_100a CUDA kernels behind the
C ABI `include/mfadd_b200.h` (libmfadd_b200.so, built in-tree).
"""
from .api import (BandedCollocation, BlockDim, BlockLayout, BlockState, Context, CudaError, Decomposition,  # noqa: F401
                  EpochStats, Field, InterfaceJump, InvalidArgument, KnotVector, LocalProblem, LogicError, MfaModel,
                  MfaddError, OutOfRange, PhaseTimings, RuntimeFault, SharedDofMap, SingularFitError, SolveResult,
                  Solver, SolverConfig, collocation_matrix, compression_ratio, decode, default_context, delta_width,
                  exchange_volume, find_span, fit_unconstrained, make_knot_vector, partition, solve, Comm,
                  shard_range, shard_box, shard_ctrl_rows, shard_exchange, solve_loopback, Side, eval_points, eval_deriv, eval_deriv_sided,
                  continuity_jumps, write_mfa, read_mfa, RawScalar, RawByteOrder, read_raw_grid,
                  ResidualStats, residual_error, SpanBasis, basis_funs, basis_derivs, basis_funs_batch)

__all__ = [n for n in dir() if not n.startswith("_")]
