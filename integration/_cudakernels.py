"""CUDA backend for `rhosolve.kernels` through librhosolve_b200 (C ABI).

Drop this file into the reference package as
`pkg/src/rhosolve/kernels/_cudakernels.py` and select it in
`kernels/__init__.py` (integration/install.py does both for a copy of the
package).  It provides the seam's four functions with the signatures,
ownership rules and return conventions of `_ckernels.pyx`:

    csr_matvec(nrows, row_ptr, col_idx, values, x) -> y      _ckernels.pyx:34
    lower_solve(Lp, Li, Lx, y)         in place, returns None _ckernels.pyx:53
    upper_solve(Up, Ui, Ux, y)         in place, returns None _ckernels.pyx:70
    factorize(n, Ap, Ai, Ax, q, drop_tol, fill_cap, row_norms)
        -> (Lp, Li, Lx, Up, Ui, Ux, pinv, fail_col)           _ckernels.pyx:144

Inputs are the reference's host arrays (int64 / complex128); they are copied
to the device as int32 / complex128, the kernels run on the current CUDA
stream, and results come back as fresh numpy arrays (or in place for the two
half-solves).  Matrices and factors are immutable in the reference
(sparse.py:31-36, factor.py:31-33), so their device copies are cached per
host array and reused across calls (one upload per matrix / factor, not one
per Krylov step).  All four are bit-identical to `_ckernels`.

Only torch (device memory) and ctypes are needed; the library path comes from
RHOSOLVE_B200_LIB.  There is no CPU fallback: a missing library or GPU raises.
"""
import ctypes
import os
import weakref

import numpy as np
import torch

BACKEND_NAME = "cuda"

_lib = ctypes.CDLL(os.environ.get("RHOSOLVE_B200_LIB", "librhosolve_b200.so"))
_vp, _i32, _i64, _f64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
_lib.rs_last_error.restype = ctypes.c_char_p
_lib.rs_csr_matvec.argtypes = [_i32, _i32] + [_vp] * 6
_lib.rs_lower_solve.argtypes = [_i32, _i32, _vp, _vp, _vp, _i64, _vp, _vp]
_lib.rs_upper_solve.argtypes = [_i32, _i32, _vp, _vp, _vp, _i64, _vp, _vp]
_lib.rs_factorize.argtypes = ([_i32, _i32, _vp, _vp, _vp, _vp, _f64, _i32, _vp, _vp, _vp, _vp,
                               _vp, _i64, _vp, _vp, _vp, _i64, _vp, _vp, _vp])
if not torch.cuda.is_available():
    raise ImportError("the cuda kernel backend needs a CUDA device")

_DEV = torch.device("cuda")
_cache = {}


def _p(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _check(rc):
    if rc != 0:
        raise RuntimeError(_lib.rs_last_error().decode())


def _upload(a, dtype):
    return torch.from_numpy(np.ascontiguousarray(a).astype(dtype, copy=False)).to(_DEV)


def _resident(a, dtype):
    """Device copy of an immutable host array, cached for the array's
    lifetime."""
    a = np.asarray(a)
    key = (id(a), a.ctypes.data, a.shape[0], np.dtype(dtype).str)
    hit = _cache.get(key)
    if hit is not None:
        return hit
    t = _upload(a, dtype)
    try:
        weakref.finalize(a, _cache.pop, key, None)
        _cache[key] = t
    except TypeError:  # not weak-referenceable (a memoryview base): no caching
        pass
    return t


def csr_matvec(nrows, row_ptr, col_idx, values, x):
    rp, ci = _resident(row_ptr, np.int32), _resident(col_idx, np.int32)
    v = _resident(values, np.complex128)
    xd = _upload(x, np.complex128)
    y = torch.empty(nrows, dtype=torch.complex128, device=_DEV)
    _check(_lib.rs_csr_matvec(1, nrows, _p(rp), _p(ci), _p(v), _p(xd), _p(y), None))
    return y.cpu().numpy()


def _half(fn, cp, ci, cx, y):
    n = len(cp) - 1
    yd = _upload(y, np.complex128)
    _check(fn(1, n, _p(_resident(cp, np.int32)), _p(_resident(ci, np.int32)),
              _p(_resident(cx, np.complex128)), len(cx), _p(yd), None))
    np.asarray(y)[:] = yd.cpu().numpy()  # the seam mutates y in place


def lower_solve(Lp, Li, Lx, y):
    _half(_lib.rs_lower_solve, Lp, Li, Lx, y)


def upper_solve(Up, Ui, Ux, y):
    _half(_lib.rs_upper_solve, Up, Ui, Ux, y)


def factorize(n, Ap, Ai, Ax, q, drop_tol, fill_cap, row_norms):
    ap, ai, ax = _upload(Ap, np.int32), _upload(Ai, np.int32), _upload(Ax, np.complex128)
    qd = _upload(q, np.int32) if q is not None else None
    rn = _upload(row_norms, np.float64) if row_norms is not None else None
    # with a cap, nnz(L) + nnz(U) <= n * cap (_ckernels.pyx:286-322); without
    # one the buffers grow by doubling, resuming where the kernel stopped
    cap = max(8 * len(Ax), 2 * n, 16) if fill_cap < 0 else n * max(fill_cap - 1, 1)
    cap = max(cap, n)
    Lp = torch.zeros(n + 1, dtype=torch.int32, device=_DEV)
    Up = torch.zeros_like(Lp)
    Li = torch.empty(cap, dtype=torch.int32, device=_DEV)
    Ui = torch.empty_like(Li)
    Lx = torch.empty(cap, dtype=torch.complex128, device=_DEV)
    Ux = torch.empty_like(Lx)
    pinv = torch.empty(n, dtype=torch.int32, device=_DEV)
    state = torch.zeros(3, dtype=torch.int32, device=_DEV)
    while True:
        _check(_lib.rs_factorize(1, n, _p(ap), _p(ai), _p(ax), _p(qd), float(drop_tol),
                                 int(fill_cap), None, _p(rn), _p(Lp), _p(Li), _p(Lx), cap,
                                 _p(Up), _p(Ui), _p(Ux), cap, _p(pinv), _p(state), None))
        s = state.cpu().numpy()
        if s[0] != 3:  # 3 = out of capacity: grow and resume
            break
        Li, Ui = (torch.cat([t, torch.empty_like(t)]) for t in (Li, Ui))
        Lx, Ux = (torch.cat([t, torch.empty_like(t)]) for t in (Lx, Ux))
        cap *= 2
    fail = int(s[1]) if s[0] == 2 else -1  # the reference's fail_col convention
    if fail >= 0:  # the reference returns whatever was built; callers only read fail_col
        lnnz = unnz = 0
    else:
        lnnz, unnz = int(Lp[-1]), int(Up[-1])

    def host(t, k, dt):
        return t[:k].cpu().numpy().astype(dt)

    return (host(Lp, n + 1, np.int64), host(Li, lnnz, np.int64), host(Lx, lnnz, np.complex128),
            host(Up, n + 1, np.int64), host(Ui, unnz, np.int64), host(Ux, unnz, np.complex128),
            host(pinv, n, np.int64), fail)
