"""ctypes binding of the C ABI in include/rhosolve_b200.h.

The library is the product: there is no Python or CPU fallback.  Importing
this module only loads the shared object; calling into it needs a CUDA device.
A missing library raises immediately with the build command.
"""

from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RHOSOLVE_B200_LIB") or os.path.join(_HERE, "_lib",
                                                               "librhosolve_b200.so")

# status codes (include/rhosolve_b200.h)
RS_OK = 0
ERRORS = {
    -1: "invalid argument",
    -2: "CUDA error",
    -3: "allocation failure",
    -4: "breakdown",
    -5: "non-finite values",
    -6: "capacity overflow",
    -7: "unsupported",
    -8: "structurally singular",
}
RS_ERR_STRUCT_SINGULAR = -8

# rs_solve_mode
INV_DIRECT, INV_BICGSTAB, INV_GMRES, LIN_DIRECT, LIN_BICGSTAB, LIN_GMRES = range(6)
# rs_solve_status
(SOLVE_OK, SOLVE_INNER_BREAKDOWN, SOLVE_INNER_NONFINITE, SOLVE_INNER_NO_PROGRESS,
 SOLVE_UNUSABLE_VECTOR, SOLVE_POWER_NOT_CONVERGED, SOLVE_SKIPPED) = range(7)
# factorize state codes
FAC_RUNNING, FAC_DONE, FAC_ZERO_PIVOT, FAC_OVERFLOW = range(4)

_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_f64 = ctypes.c_double


class SolveStats(ctypes.Structure):
    _fields_ = [("status", _i32), ("outer", _i32), ("inner_last", _i32),
                ("inner_total", _i32), ("converged", _i32), ("breakdown", _i32),
                ("final_residual", _f64), ("condest", _f64)]


STATS_BYTES = ctypes.sizeof(SolveStats)


class SolverArgs(ctypes.Structure):
    _fields_ = [("n", _i32), ("nsys", _i32), ("mode", _i32), ("threads", _i32),
                ("A_rp", _vp), ("A_ci", _vp), ("A_v", _vp),
                ("P_rp", _vp), ("P_ci", _vp), ("P_v", _vp),
                ("L_rp", _vp), ("L_ci", _vp), ("L_v", _vp),
                ("U_rp", _vp), ("U_ci", _vp), ("U_v", _vp), ("rdiag", _vp),
                ("pinv", _vp), ("rhs", _vp), ("x", _vp), ("stats", _vp),
                ("tol", _f64), ("max_iter", _i32), ("restart_m", _i32),
                ("max_outer", _i32), ("want_condest", _i32),
                ("Ls_rowoff", _vp), ("Ls_idx", _vp), ("Ls_val", _vp), ("Ls_meta", _vp),
                ("Us_rowoff", _vp), ("Us_idx", _vp), ("Us_val", _vp), ("Us_meta", _vp),
                ("Us_rd", _vp), ("colp", _vp), ("skip", _vp),
                ("trace", _vp), ("trace_count", _vp), ("trace_cap", _i32),
                ("col_reach", _i32)]


class TriFactor(ctypes.Structure):
    _fields_ = [("order", _vp), ("sptr", _vp), ("sci", _vp), ("sv", _vp), ("skey", _vp),
                ("nslices", _i32),
                ("lanes_per_row", _i32), ("active_warps", _i32), ("reserved", _i32)]


class GridArgs(ctypes.Structure):
    _fields_ = [("n", _i32), ("nb", _i32), ("mode", _i32), ("want_condest", _i32),
                ("A_rp", _vp), ("A_ci", _vp), ("A_v", _vp),
                ("P_rp", _vp), ("P_ci", _vp), ("P_v", _vp),
                ("L", TriFactor), ("U", TriFactor), ("rdiag", _vp), ("pinv", _vp),
                ("colp", _vp), ("rhs", _vp), ("x", _vp), ("stats", _vp), ("tol", _f64),
                ("max_iter", _i32), ("restart_m", _i32), ("max_outer", _i32),
                ("reserved", _i32)]


# name -> argtypes; every function returns int32 status
_SIGS = {
    "rs_abi_version": [],
    "rs_csr_matvec": [_i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp],
    "rs_factorize": [_i32, _i32, _vp, _vp, _vp, _vp, _f64, _i32, _vp, _vp, _vp, _vp, _vp,
                     _i64, _vp, _vp, _vp, _i64, _vp, _vp, _vp],
    "rs_factorize_opts": [_i32, _i32, _vp, _vp, _vp, _vp, _f64, _i32, _vp, _vp, _vp, _vp, _vp,
                           _i64, _vp, _vp, _vp, _i64, _vp, _vp, _f64, _i32, _vp],
    "rs_factor_rows": [_i32, _i32, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _i64,
                       _vp, _vp, _vp, ctypes.POINTER(_i64), _vp, _vp, _vp, _vp,
                       ctypes.POINTER(_i64), _vp],
    "rs_sell_build": [_i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "rs_pivot_recip": [_i32, _i32, _vp, _vp, _i64, _vp, _vp],
    "rs_col_sweep_supported": [_i32],
    "rs_col_stream_build": [_i32, _i32, _i32, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp,
                            _vp, ctypes.POINTER(_i64), _vp],
    "rs_lu_solve_cols": [_i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                         _vp, _vp],
    "rs_lu_solve_cols_reach": [_i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                               _vp, _i32, _vp],
    "rs_lu_solve": [_i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "rs_tri_levels": [_i32, _i32, _i32, _vp, _vp, _vp, _i64, _vp, ctypes.POINTER(_i64), _vp],
    "rs_tri_order": [_i32, _i32, _vp, _vp, _i64, _i32, _vp, ctypes.POINTER(_i64), _vp],
    "rs_tri_sell": [_i32, _i32, _i32, _vp, _vp, _vp, _vp, _i64, _i32, _vp, _vp, _vp, _vp, _vp,
                    ctypes.POINTER(_i64), _vp],
    "rs_grid_solve": [ctypes.POINTER(GridArgs), _vp],
    "rs_grid_apply": [ctypes.POINTER(GridArgs), _vp],
    "rs_lower_solve": [_i32, _i32, _vp, _vp, _vp, _i64, _vp, _vp],
    "rs_upper_solve": [_i32, _i32, _vp, _vp, _vp, _i64, _vp, _vp],
    "rs_liouvillian": [_i32, _vp, _vp, _vp, _i64, _i32, _vp, _vp, _vp, _vp,
                       ctypes.POINTER(_f64), _vp, _vp, _vp, ctypes.POINTER(_i64), _vp],
    "rs_liouvillian_batch": [_i32, _i32, _vp, _vp, _vp, _i64, _i32, _vp, _vp, _vp, _vp,
                             ctypes.POINTER(_f64), _vp, _vp, _vp, ctypes.POINTER(_i64), _vp],
    "rs_shift": [_i32, _i32, _vp, _vp, _vp, _f64, _vp, _vp, _vp, ctypes.POINTER(_i64), _vp],
    "rs_default_weight": [_i32, _i32, _vp, _vp, _vp, _i32, _vp, _vp],
    "rs_trace_modify": [_i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                        ctypes.POINTER(_i64), _vp],
    "rs_rcm": [_i32, _i32, _vp, _vp, _vp, _vp, _vp],
    "rs_same_pattern": [_i32, _i32, _vp, _vp, _i64, _vp, _vp],
    "rs_weighted_mbm_host": [_i64, _vp, _vp, _vp, _vp],
    "rs_col_min_degree_host": [_i64, _vp, _vp, _vp],
    "rs_permute": [_i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "rs_permute_rows_cols": [_i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "rs_permute_vector": [_i32, _i32, _vp, _vp, _vp, _i32, _vp],
    "rs_transpose": [_i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "rs_row_norms": [_i32, _i32, _vp, _vp, _vp, _vp],
    "rs_steady_solve": [ctypes.POINTER(SolverArgs), _vp],
    "rs_postprocess": [_i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "rs_vdots": [_i64, _i32, _vp, _vp, _vp, _vp],
    "rs_amax": [_i64, _vp, _vp, _vp],
    "rs_lincomb": [_i64, _i32, _vp, _vp, _vp, _vp, _vp],
    "rs_block_extract": [_i64, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, ctypes.POINTER(_i64),
                         _vp],
}

EXPORTED = tuple(_SIGS) + ("rs_last_error", "rs_launch_count", "rs_debug_frontal_taken",
                            "rs_tri_sell_keys")

_lib = None


def load():
    """Load the shared library (once).  Raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing; build it with `python __graft_entry__.py` "
            "or `make -C paper_1504_06768_b200/csrc` (no CPU fallback exists)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, args in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = _i32
    lib.rs_last_error.argtypes = []
    lib.rs_last_error.restype = ctypes.c_char_p
    lib.rs_launch_count.argtypes = []
    lib.rs_launch_count.restype = ctypes.c_longlong
    lib.rs_tri_sell_keys.argtypes = [_i64, _i64]
    lib.rs_tri_sell_keys.restype = _i64
    lib.rs_debug_frontal_taken.argtypes = []
    lib.rs_debug_frontal_taken.restype = _i32
    lib.rs_debug_compact_taken.argtypes = []
    lib.rs_debug_compact_taken.restype = _i32
    _lib = lib
    return lib


def call(name, *args):
    """Invoke rs_<name>; negative status raises RuntimeError with the message."""
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != RS_OK:
        msg = lib.rs_last_error().decode(errors="replace")
        kind = ERRORS.get(rc, f"status {rc}")
        if rc == -1:
            raise ValueError(f"{name}: {msg}")
        raise RuntimeError(f"{name}: {kind}: {msg}")
    return rc


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("rhosolve-b200 needs a CUDA device (sm_100a); "
                           "there is no CPU fallback")


def launch_count():
    """Kernels launched by the library so far in this process."""
    return int(load().rs_launch_count())


def stream_ptr(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def ptr(t):
    """Device pointer of a tensor (or None -> NULL)."""
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())
