"""Reverse Cuthill-McKee on the GPU (bit-identical to ordering.rcm,
pkg/src/rhosolve/ordering.py:82-118), the band/profile diagnostic
(ordering.py:40-59) and the 'cmd' ordering's two steps, weighted_mbm and
col_min_degree (ordering.py:121-282; host-native C++ in csrc/cmd_order.cu --
greedy sequential algorithms run once per structure)."""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .sparse import DeviceCSR, Permutation, as_host_csr

__all__ = ["rcm", "rcm_device", "shared_structure", "permute", "permute_rows_cols", "permute_vector", "BandProfile",
           "band_profile", "weighted_mbm", "col_min_degree", "StructurallySingularError",
           "cmd_plan"]


class StructurallySingularError(ValueError):
    """No perfect matching exists: some square submatrix of zeros blocks a
    zero-free diagonal (ordering.py:23-25)."""


def _mat(a):
    return a.matrix if hasattr(a, "matrix") else a


def shared_structure(M):
    """True when every system of a batch stores exactly system 0's pattern
    (same row extents and column indices; values may differ) -- the config-4
    sweep, whose instances differ only in a detuning."""
    if M.nsys <= 1 or M.nnz % M.nsys:
        return False
    same = torch.empty(1, dtype=torch.int32, device=M.values.device)
    _lib.call("rs_same_pattern", M.nsys, M.n, _lib.ptr(M.row_ptr), _lib.ptr(M.col_idx),
              int(M.nnz), _lib.ptr(same), _lib.stream_ptr())
    return bool(same.item())


def rcm_device(a):
    """(forward, inverse) int32 device tensors, nsys*n long (local indices).
    RCM depends on the pattern only, so a batch whose systems share system
    0's pattern is ordered once and the permutation replicated (the same
    bits as ordering every system)."""
    M = _mat(a)
    dev = M.values.device
    if shared_structure(M):
        per = M.nnz // M.nsys
        fwd = torch.empty(M.n, dtype=torch.int32, device=dev)
        inv = torch.empty_like(fwd)
        _lib.call("rs_rcm", 1, M.n, _lib.ptr(M.row_ptr), _lib.ptr(M.col_idx[:per]),
                  _lib.ptr(fwd), _lib.ptr(inv), _lib.stream_ptr())
        return fwd.repeat(M.nsys), inv.repeat(M.nsys)
    fwd = torch.empty(M.nsys * M.n, dtype=torch.int32, device=dev)
    inv = torch.empty_like(fwd)
    _lib.call("rs_rcm", M.nsys, M.n, _lib.ptr(M.row_ptr), _lib.ptr(M.col_idx), _lib.ptr(fwd),
              _lib.ptr(inv), _lib.stream_ptr())
    return fwd, inv


def rcm(a):
    """Permutation of the symmetrized structure (host arrays, as the
    reference returns); single system."""
    fwd, inv = rcm_device(a)
    return Permutation(fwd.cpu().numpy().astype("int64"), inv.cpu().numpy().astype("int64"))


def permute(a, fwd, inv):
    """sparse.permute(a, p, p) with device permutations (sparse.py:276-282)."""
    M = _mat(a)
    dev = M.values.device
    rp = torch.empty_like(M.row_ptr)
    ci = torch.empty_like(M.col_idx)
    v = torch.empty_like(M.values)
    _lib.call("rs_permute", M.nsys, M.n, _lib.ptr(M.row_ptr), _lib.ptr(M.col_idx),
              _lib.ptr(M.values), _lib.ptr(fwd), _lib.ptr(inv), _lib.ptr(rp), _lib.ptr(ci),
              _lib.ptr(v), _lib.stream_ptr())
    del dev
    return DeviceCSR(M.n, M.nsys, rp, ci, v)


def permute_rows_cols(a, row_inv, col_fwd):
    """sparse.permute(a, row_perm, col_perm) on the device: B[rf[i], cf[j]] =
    A[i, j] from rf^-1 and cf (int32 device, nsys*n; None = identity)."""
    M = _mat(a)
    dev = M.values.device
    ident = None
    if row_inv is None or col_fwd is None:
        ident = torch.arange(M.n, dtype=torch.int32, device=dev).repeat(M.nsys)
    row_inv = ident if row_inv is None else row_inv
    col_fwd = ident if col_fwd is None else col_fwd
    rp = torch.empty_like(M.row_ptr)
    ci = torch.empty_like(M.col_idx)
    v = torch.empty_like(M.values)
    _lib.call("rs_permute_rows_cols", M.nsys, M.n, _lib.ptr(M.row_ptr), _lib.ptr(M.col_idx),
              _lib.ptr(M.values), _lib.ptr(row_inv), _lib.ptr(col_fwd), _lib.ptr(rp),
              _lib.ptr(ci), _lib.ptr(v), _lib.stream_ptr())
    return DeviceCSR(M.n, M.nsys, rp, ci, v)


def permute_vector(x, fwd, nsys, n, gather):
    out = torch.empty_like(x)
    _lib.call("rs_permute_vector", nsys, n, _lib.ptr(x), _lib.ptr(fwd), _lib.ptr(out),
              1 if gather else 0, _lib.stream_ptr())
    return out


@dataclass(frozen=True)
class BandProfile:
    ub: int
    lb: int
    bandwidth: int
    up: int
    lp: int
    profile: int


def band_profile(a):
    """Upper/lower bandwidth and profile of system 0 (ordering.py:40-59)."""
    M = _mat(a)
    if M.nnz == 0:
        raise ValueError("band_profile of an empty matrix")
    n = M.n
    rp = M.row_ptr[: n + 1].long()
    cols = M.col_idx[: int(rp[-1])].long()
    rows = torch.repeat_interleave(torch.arange(n, device=cols.device), rp.diff())
    per_row = torch.zeros(n, dtype=torch.int64, device=cols.device)
    per_row.scatter_reduce_(0, rows, cols - rows, reduce="amax", include_self=True)
    per_col = torch.zeros(n, dtype=torch.int64, device=cols.device)
    per_col.scatter_reduce_(0, cols, rows - cols, reduce="amax", include_self=True)
    ub, lb = int(per_row.max()), int(per_col.max())
    up, lp = int(per_row.sum()), int(per_col.sum())
    return BandProfile(ub=ub, lb=lb, bandwidth=ub + lb + 1, up=up, lp=lp, profile=up + lp)


def _host_square(a, what):
    h = as_host_csr(_mat(a))
    if h.nrows != h.ncols:
        raise ValueError(f"{what} expects a square matrix")
    return h


def _np_ptr(x):
    return x.ctypes.data_as(ctypes.c_void_p)


def weighted_mbm(a):
    """Row permutation giving a zero-free structural diagonal
    (ordering.weighted_mbm, ordering.py:121-218): forward[r] = position of
    row r.  Raises StructurallySingularError when none exists."""
    h = _host_square(a, "weighted_mbm")
    n = h.nrows
    fwd = np.empty(n, dtype=np.int64)
    lib = _lib.load()
    rc = lib.rs_weighted_mbm_host(n, _np_ptr(h.row_ptr), _np_ptr(h.col_idx),
                                  _np_ptr(h.values), _np_ptr(fwd))
    if rc == _lib.RS_ERR_STRUCT_SINGULAR:
        raise StructurallySingularError("matrix is structurally singular: no zero-free diagonal")
    if rc != _lib.RS_OK:
        raise RuntimeError(f"rs_weighted_mbm_host: {lib.rs_last_error().decode()}")
    return Permutation(fwd)


def col_min_degree(a):
    """Exact greedy minimum-degree column ordering on the column-intersection
    graph, ties to the lowest column (ordering.col_min_degree,
    ordering.py:221-282)."""
    h = _host_square(a, "col_min_degree")
    n = h.nrows
    order = np.empty(n, dtype=np.int64)
    _lib.call("rs_col_min_degree_host", n, _np_ptr(h.row_ptr), _np_ptr(h.col_idx),
              _np_ptr(order))
    return Permutation.from_order(order)


def cmd_plan(a):
    """The 'cmd' ordering of every system of a (batch) matrix, as steady._prepare
    builds it (steady.py:95-107): weighted MBM rows when the diagonal is not
    fully stored, then column minimum degree of the row-permuted matrix.
    Returns (row_fwd, row_inv, col_fwd, col_inv) as int32 device tensors
    (nsys*n; row maps None when no system needed MBM) and the label."""
    M = _mat(a)
    B, n = M.nsys, M.n
    dev = M.values.device
    rf = np.tile(np.arange(n, dtype=np.int64), B)
    ri = rf.copy()
    cf = np.empty(B * n, dtype=np.int64)
    ci = np.empty(B * n, dtype=np.int64)
    mbm = False
    for b in range(B):
        h = M.system(b) if isinstance(M, DeviceCSR) else as_host_csr(M)
        if h.diagonal_stored_count() < n:
            p = weighted_mbm(h)
            rows, cols, vals = h.to_coo()
            h = type(h).from_coo(n, n, p.forward[rows], cols, vals, prune=False)
            rf[b * n:(b + 1) * n], ri[b * n:(b + 1) * n] = p.forward, p.inverse
            mbm = True
        c = col_min_degree(h)
        cf[b * n:(b + 1) * n], ci[b * n:(b + 1) * n] = c.forward, c.inverse

    def up(x):
        return torch.from_numpy(x.astype(np.int32)).to(dev)

    rows = (up(rf), up(ri)) if mbm else (None, None)
    return rows + (up(cf), up(ci)), ("cmd+mbm" if mbm else "cmd")
