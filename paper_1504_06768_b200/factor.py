"""Sparse LU / ILUTP on the GPU and the preconditioner apply.

Drop-in for the reference factor module (pkg/src/rhosolve/factor.py):
`lu`, `ilutp`, `solve_lu`, `condest`, `LUFactors`, `SingularMatrixError`,
`PreconditionerBreakdownError`, same argument checks and messages.  The
factorization itself is the column-pipelined kernel in csrc/ilu.cu, the apply
the reference's own column-oriented triangular solves run on shared memory
(csrc/colsweep.cuh; row-oriented sweeps in csrc/cta_ops.cuh for systems too
large for one CTA's shared memory); all are bit-identical to the reference
kernels.
"""

from __future__ import annotations

import ctypes
import math
import os

import numpy as np
import torch

from . import _lib
from .sparse import CSRMatrix, DeviceCSR, Permutation, write_matrix_market

__all__ = ["LUFactors", "lu", "ilutp", "solve_lu", "condest", "SingularMatrixError",
           "PreconditionerBreakdownError", "factor_batch", "export_factors"]


class SingularMatrixError(ValueError):
    """Complete factorization hit a zero pivot column."""


class PreconditionerBreakdownError(ValueError):
    """Incomplete factorization hit a zero pivot; retry with a smaller drop
    tolerance."""


class LUFactors:
    """P_r A = L U (approximately when incomplete) for nsys systems.

    raw:  per-system CSC exactly as the reference factorize returns it
          (Lp, Li, Lx, Up, Ui, Ux with L rows in pivotal order), pinv.
    rows: strictly-lower L and strictly-upper U in CSR + recipc(U_kk), the
          form the device triangular solves consume.
    fail: per-system zero-pivot step (-1 = ok)."""

    __slots__ = ("n", "nsys", "raw", "capL", "capU", "pinv", "L_rp", "L_ci", "L_v", "U_rp",
                 "U_ci", "U_v", "rdiag", "fill_factors", "complete", "drop_tol",
                 "fill_limit", "fail", "lnnz", "unnz", "ok", "csc", "Ls", "Us", "colp",
                 "colp_dev", "fail_dev", "solvable", "Llev", "Ulev", "nfloor", "reach")

    def ensure_cols(self):
        """Column streams of L and U for the one-CTA column sweeps
        (csrc/colsweep.cuh), built once."""
        if self.Ls is None and self.solvable:
            Lp, Li, Lx, Up, Ui, Ux = self.raw
            dev = self.pinv.device
            self.Ls = _col_stream(self.nsys, self.n, 0, Lp, Li, Lx, self.capL, None, dev)
            self.Us = _col_stream(self.nsys, self.n, 1, Up, Ui, Ux, self.capU, self.rdiag, dev)
            if self.nsys == 1 and self.ok:
                # the factors' bandwidth in pivotal coordinates: what a column
                # can touch (sliding-window sweeps of large lone systems)
                n = self.n
                cols = torch.arange(n, device=dev, dtype=torch.int32)
                lc = torch.repeat_interleave(cols, Lp[:n + 1].diff())
                uc = torch.repeat_interleave(cols, Up[:n + 1].diff())
                rl = int((Li[:lc.numel()] - lc).abs().max().item()) if lc.numel() else 0
                ru = int((Ui[:uc.numel()] - uc).abs().max().item()) if uc.numel() else 0
                self.reach = max(rl, ru, 1)
        return self

    def ensure_rows(self):
        """Build the row-oriented factor copy (row sweeps, exports) once."""
        if self.L_rp is None and self.ok:
            _build_rows(self, self.pinv.device)
        return self

    def ensure_levels(self):
        """Level-ordered copies of L and U for the grid-wide sweeps
        (csrc/levels.cu, csrc/trisell.cuh), built once."""
        if self.Llev is None and self.ok:
            self.ensure_rows()
            self.Llev = _tri_levels(self, False)
            self.Ulev = _tri_levels(self, True)
        return self

    @property
    def fill_factor(self):
        return float(self.fill_factors[0])

    def _host_csr(self, b, upper):
        """factor._csc_to_csr_matrix (factor.py:59-67): system b's L (unit
        diagonal) or U (with pivots) as a host CSR, rows in ascending column
        order (stable by the column scan)."""
        lp, li, lx, up, ui, ux, _ = self.system_raw(b)
        cp, ci, cx = (up, ui, ux) if upper else (lp, li, lx)
        n = self.n
        order = np.argsort(ci, kind="stable")
        cols = np.repeat(np.arange(n, dtype=np.int64), np.diff(cp))[order]
        rp = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(np.bincount(ci[order], minlength=n), out=rp[1:])
        return CSRMatrix(n, n, rp, cols, cx[order])

    @property
    def L(self):
        """Host CSR L of system 0 (LUFactors.L, factor.py:27-56)."""
        return self._host_csr(0, False)

    @property
    def U(self):
        """Host CSR U of system 0 (LUFactors.U)."""
        return self._host_csr(0, True)

    @property
    def row_perm(self):
        """Permutation(pinv) of system 0 (LUFactors.row_perm)."""
        return Permutation(self.pinv[: self.n].cpu().numpy().astype(np.int64))

    @property
    def col_perm(self):
        """Column pre-ordering (LUFactors.col_perm): the 'cmd' minimum-degree
        order when one was given, else the identity."""
        return self.colp if self.colp is not None else Permutation.identity(self.n)

    def system_raw(self, b):
        """Host copy of system b's raw CSC factors (reference layout, int64)."""
        Lp, Li, Lx, Up, Ui, Ux = self.raw
        n = self.n
        lp = Lp[b * (n + 1):(b + 1) * (n + 1)].cpu().numpy().astype(np.int64)
        up = Up[b * (n + 1):(b + 1) * (n + 1)].cpu().numpy().astype(np.int64)
        li = Li[b * self.capL:b * self.capL + lp[-1]].cpu().numpy().astype(np.int64)
        lx = Lx[b * self.capL:b * self.capL + lp[-1]].cpu().numpy()
        ui = Ui[b * self.capU:b * self.capU + up[-1]].cpu().numpy().astype(np.int64)
        ux = Ux[b * self.capU:b * self.capU + up[-1]].cpu().numpy()
        pinv = self.pinv[b * n:(b + 1) * n].cpu().numpy().astype(np.int64)
        return lp, li, lx, up, ui, ux, pinv

    def __repr__(self):
        kind = "complete" if self.complete else "incomplete"
        return f"LUFactors(n={self.n}, nsys={self.nsys}, {kind}, fill={self.fill_factors})"


def _transpose(M):
    rp = torch.empty_like(M.row_ptr)
    ci = torch.empty_like(M.col_idx)
    v = torch.empty_like(M.values)
    _lib.call("rs_transpose", M.nsys, M.n, _lib.ptr(M.row_ptr), _lib.ptr(M.col_idx),
              _lib.ptr(M.values), _lib.ptr(rp), _lib.ptr(ci), _lib.ptr(v), _lib.stream_ptr())
    return rp, ci, v


def factor_batch(M, drop_tol, fill_limit, raise_on_fail=True, capacity=None, eager=True,
                 pivot_floor=0.0, early_drop=False):
    """factor._factor (factor.py:70-112) for every system of a DeviceCSR.
    pivot_floor > 0 switches on the zero-pivot substitution of
    rs_factorize_opts (NOT reference behaviour; block-Jacobi blocks only);
    LUFactors.nfloor then counts the substituted pivots per system; early_drop
    is the Saad-ILUT rule (drop a U entry before eliminating with it)."""
    n, B = M.n, M.nsys
    dev = M.values.device
    if n == 0 or M.nnz == 0:
        raise SingularMatrixError("zero pivot at elimination step 0")
    incomplete = drop_tol > 0.0 or not math.isinf(fill_limit)
    # entries per system: the row pointer at the system boundaries (one strided read)
    nnz_rows = np.diff(M.row_ptr[::n].cpu().numpy().astype(np.int64))
    if math.isinf(fill_limit):
        cap = -1
    else:
        # per-system cap (factor.py:92); systems of a batch share n and, in
        # every configuration, nnz -- a differing nnz would change the cap.
        caps = [int(math.ceil(fill_limit * int(z) / n)) for z in nnz_rows]
        cap = max(caps)
    caps_t = None
    if cap >= 0 and len(set(caps)) > 1:  # per-system caps (e.g. block-Jacobi blocks)
        caps_t = torch.tensor(caps, dtype=torch.int32, device=dev)
    Ap, Ai, Ax = _transpose(M)
    rn = None
    if drop_tol > 0.0:
        rn = torch.empty(B * n, dtype=torch.float64, device=dev)
        _lib.call("rs_row_norms", B, n, _lib.ptr(M.row_ptr), _lib.ptr(M.values), _lib.ptr(rn),
                  _lib.stream_ptr())
    maxnnz = int(nnz_rows.max())
    per_col = max(cap - 1, 1) if cap >= 0 else None
    guess = max(24 * maxnnz, 2 * n, 16)
    capL = capU = min(n * per_col, guess) if per_col else guess
    if capacity is not None:  # tests: force the overflow/resume path
        capL = capU = max(int(capacity), n)
    Lp = torch.zeros(B * (n + 1), dtype=torch.int32, device=dev)
    Up = torch.zeros_like(Lp)
    Li = torch.empty(B * capL, dtype=torch.int32, device=dev)
    Lx = torch.empty(B * capL, dtype=torch.complex128, device=dev)
    Ui = torch.empty(B * capU, dtype=torch.int32, device=dev)
    Ux = torch.empty(B * capU, dtype=torch.complex128, device=dev)
    pinv = torch.empty(B * n, dtype=torch.int32, device=dev)
    state = torch.zeros(3 * B, dtype=torch.int32, device=dev)
    st = _lib.stream_ptr()
    while True:
        _lib.call("rs_factorize_opts", B, n, _lib.ptr(Ap), _lib.ptr(Ai), _lib.ptr(Ax), None,
                  float(drop_tol), cap, _lib.ptr(caps_t), _lib.ptr(rn), _lib.ptr(Lp),
                  _lib.ptr(Li), _lib.ptr(Lx), capL, _lib.ptr(Up), _lib.ptr(Ui), _lib.ptr(Ux),
                  capU, _lib.ptr(pinv), _lib.ptr(state), float(pivot_floor),
                  1 if early_drop else 0, st)
        sh = state.reshape(B, 3).cpu().numpy()
        if not np.any(sh[:, 0] == 3):
            break
        # grow (x2) both factors of every system, preserving contents
        ncapL, ncapU = 2 * capL, 2 * capU
        Li, Lx = _regrow(Li, B, capL, ncapL), _regrow(Lx, B, capL, ncapL)
        Ui, Ux = _regrow(Ui, B, capU, ncapU), _regrow(Ux, B, capU, ncapU)
        capL, capU = ncapL, ncapU
    fail = np.where(sh[:, 0] == 2, sh[:, 1], -1)
    if raise_on_fail and np.any(fail >= 0):
        k = int(fail[fail >= 0][0])
        msg = f"zero pivot at elimination step {k}"
        raise PreconditionerBreakdownError(msg) if incomplete else SingularMatrixError(msg)
    f = LUFactors()
    f.n, f.nsys = n, B
    f.raw = (Lp, Li, Lx, Up, Ui, Ux)
    f.capL, f.capU = capL, capU
    f.pinv = pinv
    lp = Lp.reshape(B, n + 1)[:, -1].cpu().numpy().astype(np.int64)
    up = Up.reshape(B, n + 1)[:, -1].cpu().numpy().astype(np.int64)
    f.lnnz, f.unnz = lp, up
    f.fill_factors = (lp + up) / nnz_rows
    f.complete = not incomplete
    f.drop_tol = float(drop_tol) if incomplete else None
    f.fill_limit = float(fill_limit) if incomplete else None
    f.fail = fail
    f.nfloor = sh[:, 2].copy()
    f.ok = bool(np.all(fail < 0))
    f.L_rp = f.L_ci = f.L_v = f.U_rp = f.U_ci = f.U_v = None
    f.rdiag = None
    # the preconditioner apply consumes the raw CSC factors directly (the
    # reference's column loops) whenever the sweep vector fits shared memory;
    # larger systems use the row-oriented copy
    f.csc = bool(_lib.load().rs_col_sweep_supported(n))
    f.Ls = f.Us = None
    f.reach = 0
    f.Llev = f.Ulev = None
    f.colp = f.colp_dev = None
    # a batch with some failed systems can still be solved on the column-sweep
    # path: the solver masks the failed ones (rs_solver_args.skip)
    f.fail_dev = None if f.ok else torch.from_numpy((fail >= 0).astype(np.int32)).to(dev)
    f.solvable = f.ok or (f.csc and bool(np.any(fail < 0)))
    if f.solvable:
        f.rdiag = torch.empty(B * n, dtype=torch.complex128, device=dev)
        _lib.call("rs_pivot_recip", B, n, _lib.ptr(Up), _lib.ptr(Ux), capU,
                  _lib.ptr(f.rdiag), st)
        # the apply layouts are built on first use: column streams (one CTA
        # per system), row-oriented CSR, or level-ordered SELL (grid-wide)
        if eager and f.csc and n < grid_min_n():
            f.ensure_cols()
    return f


def grid_min_n():
    """Systems of at least this order are solved by the grid-wide kernels
    (csrc/grid.cu) instead of one CTA per system."""
    import os
    return int(os.environ.get("RHOSOLVE_GRID_MIN_N", "8192"))


COL_STREAM_WIDTH = 64  # entries per stream row (csrc/colsweep.cuh CW)


def _col_stream(B, n, upper, cp, ci, cv, cap, rdiag, dev):
    """Column stream of one triangle (csrc/colsweep.cuh): (rowoff, idx, val,
    meta, rrd)."""
    rowoff = torch.empty(B * n + 1, dtype=torch.int32, device=dev)
    rows = ctypes.c_int64(0)
    st = _lib.stream_ptr()
    _lib.call("rs_col_stream_build", B, n, upper, _lib.ptr(cp), _lib.ptr(ci), _lib.ptr(cv), cap,
              _lib.ptr(rdiag), _lib.ptr(rowoff), None, None, None, None, ctypes.byref(rows), st)
    R = max(rows.value, 1)
    idx = torch.empty(COL_STREAM_WIDTH * R, dtype=torch.int32, device=dev)
    val = torch.empty(COL_STREAM_WIDTH * R, dtype=torch.complex128, device=dev)
    meta = torch.empty(R, dtype=torch.int32, device=dev)
    rrd = torch.empty(R, dtype=torch.complex128, device=dev) if upper else None
    _lib.call("rs_col_stream_build", B, n, upper, _lib.ptr(cp), _lib.ptr(ci), _lib.ptr(cv), cap,
              _lib.ptr(rdiag), _lib.ptr(rowoff), _lib.ptr(idx), _lib.ptr(val), _lib.ptr(meta),
              _lib.ptr(rrd), ctypes.byref(rows), st)
    return rowoff, idx, val, meta, rrd


def _regrow(t, B, old, new):
    out = torch.empty(B * new, dtype=t.dtype, device=t.device)
    out.view(B, new)[:, :old].copy_(t.view(B, old))
    return out


def _build_rows(f, dev):
    B, n = f.nsys, f.n
    Lp, Li, Lx, Up, Ui, Ux = f.raw
    f.L_rp = torch.empty(B * n + 1, dtype=torch.int32, device=dev)
    f.U_rp = torch.empty_like(f.L_rp)
    ln, un = ctypes.c_int64(0), ctypes.c_int64(0)
    st = _lib.stream_ptr()
    args = lambda lci, lv, uci, uv, rd: (  # noqa: E731
        B, n, _lib.ptr(Lp), _lib.ptr(Li), _lib.ptr(Lx), f.capL, _lib.ptr(Up), _lib.ptr(Ui),
        _lib.ptr(Ux), f.capU, _lib.ptr(f.L_rp), lci, lv, ctypes.byref(ln), _lib.ptr(f.U_rp),
        uci, uv, rd, ctypes.byref(un), st)
    _lib.call("rs_factor_rows", *args(None, None, None, None, None))
    f.L_ci = torch.empty(max(ln.value, 1), dtype=torch.int32, device=dev)
    f.L_v = torch.empty(max(ln.value, 1), dtype=torch.complex128, device=dev)
    f.U_ci = torch.empty(max(un.value, 1), dtype=torch.int32, device=dev)
    f.U_v = torch.empty(max(un.value, 1), dtype=torch.complex128, device=dev)
    rd = torch.empty(B * n, dtype=torch.complex128, device=dev)
    _lib.call("rs_factor_rows", *args(_lib.ptr(f.L_ci), _lib.ptr(f.L_v), _lib.ptr(f.U_ci),
                                      _lib.ptr(f.U_v), _lib.ptr(rd)))
    f.rdiag = rd


class TriLevels:
    """One triangle in level order (csrc/levels.cu): rows sorted by dependency
    level, levels padded to whole slices of H = 32/G rows, SELL storage."""

    __slots__ = ("order", "sptr", "sci", "sv", "skey", "nslices", "G", "nlevels", "entries",
                 "apw", "level")

    def fill(self, t):
        """Populate an _lib.TriFactor."""
        t.order, t.sptr = self.order.data_ptr(), self.sptr.data_ptr()
        t.sci, t.sv, t.skey = self.sci.data_ptr(), self.sv.data_ptr(), self.skey.data_ptr()
        t.nslices, t.lanes_per_row = self.nslices, self.G
        t.active_warps = self.apw
        t.reserved = int(os.environ.get("RHOSOLVE_TRI_MODE", "0"))  # tuning hook


def _tri_levels(f, upper):
    B, n = f.nsys, f.n
    N = B * n
    dev = f.pinv.device
    rp, ci, v = (f.U_rp, f.U_ci, f.U_v) if upper else (f.L_rp, f.L_ci, f.L_v)
    st = _lib.stream_ptr()
    level = torch.empty(N, dtype=torch.int32, device=dev)
    nlev = ctypes.c_int64(0)
    Lp, Li, _, Up, Ui, _ = f.raw
    cp, ri, cap = (Up, Ui, f.capU) if upper else (Lp, Li, f.capL)
    _lib.call("rs_tri_levels", B, n, int(upper), _lib.ptr(rp), _lib.ptr(cp), _lib.ptr(ri), cap,
              _lib.ptr(level), ctypes.byref(nlev), st)
    # rows per slice: as many as a level typically holds (power of two <= 32);
    # the other 32/H lanes of a warp share each row's entries
    per_level = N / max(nlev.value, 1)
    avg_len = float(rp[-1].item()) / max(N, 1)
    if per_level >= 24:
        # wide DAG: one lane per row (two lanes per row halve the steps of a
        # slice but double the slices and their polling: measured slower on
        # config 5, 12.1 vs 7.8 ms per apply)
        H = 32
    else:
        H = 8 if per_level >= 6 else 1
    env_h = os.environ.get("RHOSOLVE_TRI_H")
    if env_h:
        H = int(env_h)
    order = torch.empty(N + H * nlev.value, dtype=torch.int32, device=dev)
    npos = ctypes.c_int64(0)
    _lib.call("rs_tri_order", B, n, _lib.ptr(level), _lib.ptr(rp), nlev.value, H,
              _lib.ptr(order), ctypes.byref(npos), st)
    nsl = npos.value // H
    sptr = torch.empty(nsl + 1, dtype=torch.int32, device=dev)
    total = ctypes.c_int64(0)
    args = (B, n, int(upper), _lib.ptr(rp), _lib.ptr(ci), _lib.ptr(v), _lib.ptr(order),
            npos.value, H, _lib.ptr(level), _lib.ptr(sptr))
    _lib.call("rs_tri_sell", *args, None, None, None, ctypes.byref(total), st)
    t = TriLevels()
    t.sci = torch.empty(max(total.value, 1), dtype=torch.int32, device=dev)
    t.sv = torch.empty(max(total.value, 1), dtype=torch.complex128, device=dev)
    nkeys = int(_lib.load().rs_tri_sell_keys(total.value, nsl))
    t.skey = torch.empty(nkeys, dtype=torch.int32, device=dev)
    _lib.call("rs_tri_sell", *args, _lib.ptr(t.sci), _lib.ptr(t.sv), _lib.ptr(t.skey),
              ctypes.byref(total), st)
    t.order, t.sptr, t.nslices, t.G = order[:npos.value], sptr, nsl, 32 // H
    t.nlevels, t.entries = nlev.value, total.value
    t.level = level  # per-row dependency level (diagnostics)
    # sweep window: enough slices in flight to cover ~16 levels of look-ahead,
    # spread over the SMs (16 warps per CTA at most; 0 = all)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    want = 16.0 * nsl / max(nlev.value, 1)
    t.apw = int(min(16, max(1, round(want / sms))))
    env = os.environ.get("RHOSOLVE_TRI_APW")
    if env:
        t.apw = int(env)
    return t


def _mat(a):
    return a.matrix if hasattr(a, "matrix") else a


def _with_colperm(M, col_perm, drop_tol, fill_limit):
    """factor._factor's column pre-ordering (factor.py:76-78): the reference
    eliminates column q[k] at step k (q = col_perm.inverse); factoring the
    column-permuted matrix A[:, q] in natural order gives the same factors
    bit for bit, and solve_lu scatters x[q] = y back."""
    if col_perm is None or col_perm.is_identity():
        return factor_batch(M, drop_tol, fill_limit)
    if len(col_perm) != M.n:
        raise ValueError("column permutation length does not match matrix")
    from . import ordering
    cf = torch.from_numpy(np.tile(col_perm.forward, M.nsys).astype(np.int32)).to(
        M.values.device)
    f = factor_batch(ordering.permute_rows_cols(M, None, cf), drop_tol, fill_limit)
    f.colp, f.colp_dev = col_perm, cf
    return f


def lu(a, col_perm=None):
    """Complete sparse LU with partial pivoting (factor.py:115-118)."""
    return _with_colperm(_mat(a), col_perm, 0.0, math.inf)


def ilutp(a, d=1e-4, p=300.0, col_perm=None):
    """ILUTP with drop tolerance d and fill budget p (factor.py:121-134)."""
    if d < 0:
        raise ValueError("drop tolerance d must be >= 0")
    if not p >= 1:
        raise ValueError("fill limit p must be >= 1")
    return _with_colperm(_mat(a), col_perm, float(d), float(p))


def solve_lu_device(f, b):
    """x = M^{-1} b on the device for every system (b: nsys*n complex128)."""
    x = _solve_lu_rows(f, b)
    if f.colp_dev is not None:  # x[q] = y (factor.py:147-148)
        y = torch.empty_like(x)
        _lib.call("rs_permute_vector", f.nsys, f.n, _lib.ptr(x), _lib.ptr(f.colp_dev),
                  _lib.ptr(y), 1, _lib.stream_ptr())
        return y
    return x


def _levels_no_colp(f, b):
    """solve_lu_levels without the final column scatter (the caller applies it)."""
    keep, f.colp_dev = f.colp_dev, None
    try:
        return solve_lu_levels(f, b)
    finally:
        f.colp_dev = keep


def solve_lu_levels(f, b):
    """x = M^{-1} b through the grid-wide level-ordered sweeps (the apply of the
    large-system solver, csrc/grid.cu); bit-identical to the column sweeps."""
    f.ensure_levels()
    x = torch.empty_like(b)
    a = _lib.GridArgs()
    a.n, a.nb = f.nsys * f.n, f.n
    f.Llev.fill(a.L)
    f.Ulev.fill(a.U)
    a.rdiag, a.pinv = f.rdiag.data_ptr(), f.pinv.data_ptr()
    if f.colp_dev is not None:
        a.colp = f.colp_dev.data_ptr()
    a.rhs, a.x = b.data_ptr(), x.data_ptr()
    _lib.call("rs_grid_apply", ctypes.byref(a), _lib.stream_ptr())
    return x


def _solve_lu_rows(f, b):
    if f.n >= grid_min_n() and f.ok and float(np.sum(f.lnnz + f.unnz)) / (f.nsys * f.n) < 64.0:
        return _levels_no_colp(f, b)  # wide DAG (steady._wide): grid-wide level sweeps
    x = torch.empty_like(b)
    if f.csc:
        f.ensure_cols()
        (lo, li, lv, lm, _), (uo, ui, uv, um, ur) = f.Ls, f.Us
        _lib.call("rs_lu_solve_cols_reach", f.nsys, f.n, _lib.ptr(f.pinv), _lib.ptr(lo),
                  _lib.ptr(li), _lib.ptr(lv), _lib.ptr(lm), _lib.ptr(uo), _lib.ptr(ui),
                  _lib.ptr(uv), _lib.ptr(um), _lib.ptr(ur), _lib.ptr(b), _lib.ptr(x),
                  int(f.reach), _lib.stream_ptr())
        return x
    f.ensure_rows()
    _lib.call("rs_lu_solve", f.nsys, f.n, _lib.ptr(f.pinv), _lib.ptr(f.L_rp), _lib.ptr(f.L_ci),
              _lib.ptr(f.L_v), _lib.ptr(f.U_rp), _lib.ptr(f.U_ci), _lib.ptr(f.U_v),
              _lib.ptr(f.rdiag), _lib.ptr(b), _lib.ptr(x), _lib.stream_ptr())
    return x


def solve_lu(f, b):
    """factor.solve_lu (factor.py:137-149).  numpy in -> numpy out; a CUDA
    tensor in -> CUDA tensor out."""
    if isinstance(b, torch.Tensor):
        return solve_lu_device(f, b.to(torch.complex128).contiguous())
    b = np.asarray(b, dtype=np.complex128)
    if b.shape != (f.n * f.nsys,):
        raise ValueError(f"rhs length {b.shape} does not match n={f.n}")
    dev = f.pinv.device
    return solve_lu_device(f, torch.from_numpy(b).to(dev)).cpu().numpy()


def condest(f):
    """||M^{-1} 1||_inf (factor.py:152-157); one value per system."""
    e = torch.ones(f.nsys * f.n, dtype=torch.complex128, device=f.pinv.device)
    x = solve_lu_device(f, e).reshape(f.nsys, f.n).abs().amax(1).cpu().numpy()
    return float(x[0]) if f.nsys == 1 else x


def export_factors(f, prefix):
    """Write L/U as Matrix Market files and the permutations as
    newline-delimited integer lists: <prefix>_L.mtx, _U.mtx, _rowperm.txt,
    _colperm.txt (factor.py:160-167); system 0 of a batch."""
    write_matrix_market(f.L, f"{prefix}_L.mtx")
    write_matrix_market(f.U, f"{prefix}_U.mtx")
    f.row_perm.save(f"{prefix}_rowperm.txt")
    f.col_perm.save(f"{prefix}_colperm.txt")
