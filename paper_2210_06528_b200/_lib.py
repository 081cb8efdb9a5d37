"""ctypes loader for libmfadd_b200.so (the C ABI in include/mfadd_b200.h).

There is no fallback: if the library is missing or fails to load, importing
the product API raises.  The library is built in-tree by
`paper_2210_06528_b200.build.build()` (or `__graft_entry__.build()`).
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# MFADD_DEBUG=1 selects the bounds-checked build (libmfadd_b200_debug.so)
LIB_PATH = os.path.join(HERE, "libmfadd_b200_debug.so" if os.environ.get("MFADD_DEBUG") else "libmfadd_b200.so")
if os.environ.get("MFADD_LIB_VARIANT"):  # measurement aid: an in-tree build variant (libmfadd_b200_<v>.so)
    LIB_PATH = os.path.join(HERE, f"libmfadd_b200_{os.environ['MFADD_LIB_VARIANT']}.so")

c_dp = C.POINTER(C.c_double)
c_lp = C.POINTER(C.c_int64)
c_ip = C.POINTER(C.c_int)

MFADD_OK, MFADD_EINVAL, MFADD_ERANGE, MFADD_ESINGULAR, MFADD_ERUNTIME, MFADD_ELOGIC, MFADD_ECUDA, MFADD_ENOMEM = \
    range(8)


class SolverConfigC(C.Structure):
    _fields_ = [("max_outer_iterations", C.c_int), ("tolerance", C.c_double), ("workers", C.c_int),
                ("log_errors", C.c_int), ("enforce_continuity", C.c_int), ("store_error", C.c_int)]


class SolveSummaryC(C.Structure):
    _fields_ = [("converged", C.c_int), ("constraint_iterations", C.c_int), ("n_epochs", C.c_int),
                ("n_final_jumps", C.c_int), ("final_dp", C.c_double), ("global_l2", C.c_double),
                ("global_linf", C.c_double), ("t_setup", C.c_double), ("t_local_solve", C.c_double),
                ("t_exchange", C.c_double), ("t_constraint", C.c_double), ("t_decode", C.c_double)]


class ModelViewC(C.Structure):
    _fields_ = [("rank", C.c_int), ("degrees", c_ip), ("clamp_left", C.POINTER(C.c_ubyte)),
                ("clamp_right", C.POINTER(C.c_ubyte)), ("knots", c_dp), ("kn_off", c_lp), ("ctrl_ext", c_lp),
                ("bounds", c_dp), ("nprov", C.c_int), ("prov_keys", C.POINTER(C.c_char_p)),
                ("prov_values", C.POINTER(C.c_char_p)), ("controls", c_dp)]


class EpochStatsC(C.Structure):
    _fields_ = [("iteration", C.c_int), ("dp_max", C.c_double), ("jump_ss", C.c_double), ("jump_ms", C.c_double)]


# name -> (restype, argtypes); argtypes None = left unchecked (pointers)
_SIGS = {
    "mfadd_abi_version": (C.c_int, []),
    "mfadd_last_error": (C.c_char_p, []),
    "mfadd_last_error_dim": (C.c_int, []),
    "mfadd_last_error_span": (C.c_int64, []),
    "mfadd_partition": (C.c_int, [C.c_int, c_lp, c_dp, c_ip, C.c_int, c_lp, C.c_int64, C.c_int,
                                  C.POINTER(C.c_void_p)]),
    "mfadd_decomposition_free": (None, [C.c_void_p]),
    "mfadd_dec_rank": (C.c_int, [C.c_void_p]),
    "mfadd_dec_block_count": (C.c_int, [C.c_void_p]),
    "mfadd_dec_block_dims": (None, [C.c_void_p, c_lp]),
    "mfadd_dec_coords": (None, [C.c_void_p, c_ip]),
    "mfadd_dec_nctrl": (None, [C.c_void_p, c_lp]),
    "mfadd_dec_knots": (C.c_int, [C.c_void_p, C.c_int, c_dp]),
    "mfadd_dec_neighbors": (C.c_int, [C.c_void_p, C.c_int, c_ip, C.c_int]),
    "mfadd_dec_holder_ranges": (None, [C.c_void_p, C.c_int, c_ip]),
    "mfadd_dec_exchange_volume": (None, [C.c_void_p, c_lp]),
    "mfadd_dec_compression_ratio": (C.c_double, [C.c_void_p]),
    "mfadd_dec_any_shared": (C.c_int, [C.c_void_p]),
    "mfadd_dec_grid_dims": (None, [C.c_void_p, c_lp]),
    "mfadd_context_create": (C.c_int, [C.c_int, C.c_void_p, C.POINTER(C.c_void_p)]),
    "mfadd_context_free": (None, [C.c_void_p]),
    "mfadd_context_launch_count": (C.c_int64, [C.c_void_p]),
    "mfadd_solver_create": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(SolverConfigC), C.POINTER(C.c_void_p)]),
    "mfadd_solver_free": (None, [C.c_void_p]),
    "mfadd_solve": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.POINTER(SolveSummaryC)]),
    "mfadd_solve_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(SolveSummaryC)]),
    "mfadd_solve_host_batch": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                         C.POINTER(SolveSummaryC)]),
    "mfadd_solver_epochs": (C.c_int, [C.c_void_p, C.POINTER(EpochStatsC), C.c_int]),
    "mfadd_solver_final_jumps": (C.c_int, [C.c_void_p, c_dp, C.c_int]),
    "mfadd_solver_controls": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int]),
    "mfadd_solver_global_error": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int]),
    "mfadd_solver_block_controls": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_int]),
    "mfadd_solver_block_errors": (C.c_int, [C.c_void_p, C.c_int, c_dp]),
    "mfadd_solver_device_controls": (C.c_void_p, [C.c_void_p]),
    "mfadd_solver_last_launches": (C.c_int, [C.c_void_p]),
    "mfadd_solver_set_profiling": (C.c_int, [C.c_void_p, C.c_int]),
    "mfadd_solver_kernel_times": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int, c_dp, C.c_int]),
    "mfadd_collocation": (C.c_int, [C.c_void_p, c_dp, C.c_int, C.c_int, c_dp, C.c_int64, C.c_int64, C.c_int64,
                                    c_lp, c_ip, c_dp]),
    "mfadd_fit_unconstrained": (C.c_int, [C.c_void_p, C.c_int, C.c_int, c_dp, c_lp, c_dp, c_lp, c_lp, c_lp, c_dp,
                                          c_dp]),
    "mfadd_residual_error": (C.c_int, [C.c_void_p, C.c_int, C.c_int, c_dp, c_lp, c_dp, c_lp, c_lp, c_lp, c_dp, c_dp,
                                       c_dp, c_dp, c_dp]),
    "mfadd_basis_funs": (C.c_int, [C.c_void_p, c_dp, C.c_int, C.c_int, C.c_int64, c_dp, c_ip, C.c_int, c_ip, c_dp]),
    "mfadd_decode": (C.c_int, [C.c_void_p, C.c_int, C.c_int, c_dp, c_lp, c_dp, c_lp, c_lp, c_lp, c_dp, c_dp]),
    "mfadd_eval_points": (C.c_int, [C.c_void_p, C.c_int, c_ip, c_dp, c_lp, c_lp, c_lp, c_dp, C.c_int64, c_dp, c_ip,
                                    C.c_int, C.c_int, c_dp]),
    "mfadd_continuity_jumps": (C.c_int, [C.c_void_p, C.c_int, c_ip, c_dp, c_lp, c_lp, c_dp, C.c_int, C.c_double,
                                         C.c_int, C.c_int, c_dp]),
    "mfadd_solver_continuity_probe": (C.c_int, [C.c_void_p, C.c_int, C.c_int, c_dp, c_ip]),
    "mfadd_decode_grid": (C.c_int, [C.c_void_p, C.c_int, C.c_int, c_dp, c_lp, c_lp, c_dp, c_lp, c_dp]),
    "mfadd_write_mfa": (C.c_int, [C.c_char_p, C.POINTER(ModelViewC)]),
    "mfadd_read_mfa": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p)]),
    "mfadd_model_view_of": (C.c_int, [C.c_void_p, C.POINTER(ModelViewC)]),
    "mfadd_model_free": (None, [C.c_void_p]),
    "mfadd_read_raw_grid": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int, c_lp, C.c_int, C.c_int, C.c_void_p, C.c_int]),
    "mfadd_nccl_unique_id": (C.c_int, [C.c_void_p]),
    "mfadd_comm_create": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "mfadd_comm_free": (None, [C.c_void_p]),
    "mfadd_solver_create_sharded": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(SolverConfigC), C.c_void_p,
                                              C.POINTER(C.c_void_p)]),
    "mfadd_shard_range": (C.c_int, [C.c_void_p, C.c_int, C.c_int, c_ip, c_ip, c_lp, c_lp]),
    "mfadd_shard_box": (C.c_int, [C.c_void_p, C.c_int, C.c_int, c_lp, c_lp]),
    "mfadd_shard_ctrl_rows": (C.c_int, [C.c_void_p, C.c_int, C.c_int, c_lp, c_lp]),
    "mfadd_solver_gather_controls": (C.c_int, [C.c_void_p]),
    "mfadd_shard_exchange": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, c_lp, C.c_int64]),
    "mfadd_solve_loopback": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(SolverConfigC), C.c_int, C.c_void_p,
                                       C.c_void_p, C.c_void_p, C.POINTER(SolveSummaryC), C.POINTER(EpochStatsC),
                                       C.c_int, c_dp, C.c_int]),
}

# Symbols include/mfadd_b200.h declares (checked by the CPU test suite).
EXPORTED = tuple(_SIGS)

_lib = None


def load():
    """Load the CUDA library (raises if it is absent: no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with paper_2210_06528_b200.build.build() "
                              f"(there is no CPU fallback)")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib
