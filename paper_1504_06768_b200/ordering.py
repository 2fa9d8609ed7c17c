"""Reverse Cuthill-McKee on the GPU (bit-identical to ordering.rcm,
pkg/src/rhosolve/ordering.py:82-118) and the band/profile diagnostic
(ordering.py:40-59)."""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _lib
from .sparse import DeviceCSR, Permutation

__all__ = ["rcm", "rcm_device", "permute", "permute_vector", "BandProfile", "band_profile"]


def _mat(a):
    return a.matrix if hasattr(a, "matrix") else a


def rcm_device(a):
    """(forward, inverse) int32 device tensors, nsys*n long (local indices)."""
    M = _mat(a)
    dev = M.values.device
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
