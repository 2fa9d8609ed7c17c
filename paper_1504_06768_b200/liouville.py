"""Lindblad superoperator and its solver-ready variants, assembled on the GPU.

Drop-in for the reference liouville module (pkg/src/rhosolve/liouville.py):
same function names, arguments, variants and errors; the matrix lives on the
device as a `DeviceCSR` (a block-diagonal batch when several systems are
built together).  Column-stacking convention: vec index = col*D + row.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .sparse import DeviceCSR, as_host_csr, from_host

__all__ = ["LiouvillianSystem", "build_liouvillian", "build_liouvillian_batch", "shift",
           "build_modified", "default_weight", "DEFAULT_SIGMA", "concat_systems", "on_device"]

DEFAULT_SIGMA = 1e-15
_HERM_TOL = 1e-12


class LiouvillianSystem:
    """Superoperator matrix plus Hilbert dimension and variant tag
    ("plain", "shifted" with sigma, "modified" with weight and rhs), as in
    liouville.py:21-51.  For a batch, weight is an array and rhs is
    nsys*n long."""

    __slots__ = ("matrix", "hilbert_dim", "variant", "sigma", "weight", "rhs")

    def __init__(self, matrix, hilbert_dim, variant, sigma=None, weight=None, rhs=None):
        if matrix.n != hilbert_dim * hilbert_dim:
            raise ValueError("matrix side must equal hilbert_dim squared")
        if variant not in ("plain", "shifted", "modified"):
            raise ValueError(f"unknown variant {variant!r}")
        self.matrix = matrix
        self.hilbert_dim = int(hilbert_dim)
        self.variant = variant
        self.sigma = sigma
        self.weight = weight
        self.rhs = rhs

    @property
    def n(self):
        return self.matrix.n

    @property
    def nsys(self):
        return self.matrix.nsys

    def __repr__(self):
        return (f"LiouvillianSystem(D={self.hilbert_dim}, variant={self.variant!r}, "
                f"nsys={self.nsys}, nnz={self.matrix.nnz})")


def on_device(L, device=None, values_stream=None):
    """L with its matrix resident on the GPU: a host CSRMatrix, a list-built
    batch or a PinnedBatchCSR is uploaded (pinned batches asynchronously on
    the current stream, values on `values_stream` when given -- see
    sparse.from_host); a DeviceCSR passes through unchanged."""
    if isinstance(L.matrix, DeviceCSR):
        return L
    return LiouvillianSystem(from_host(L.matrix, device, values_stream=values_stream),
                             L.hilbert_dim, L.variant, sigma=L.sigma, weight=L.weight,
                             rhs=L.rhs)


def _dev_op(m, dev):
    h = as_host_csr(m)
    return (torch.from_numpy(h.row_ptr.astype(np.int32)).to(dev),
            torch.from_numpy(h.col_idx.astype(np.int32)).to(dev),
            torch.from_numpy(np.ascontiguousarray(h.values)).to(dev), h.nnz)


def _assemble(H, collapse_ops, dev):
    D = H.matrix.nrows
    for c in collapse_ops:
        if tuple(c.dims) != tuple(H.dims):
            raise ValueError(f"collapse operator dims {c.dims} do not match H {H.dims}")
    hrp, hci, hv, hnnz = _dev_op(H.matrix, dev)
    cops = [_dev_op(c.matrix, dev) for c in collapse_ops]
    K = len(cops)
    PArr = ctypes.c_void_p * max(K, 1)
    c_rp = PArr(*[c[0].data_ptr() for c in cops])
    c_ci = PArr(*[c[1].data_ptr() for c in cops])
    c_v = PArr(*[c[2].data_ptr() for c in cops])
    c_nnz = (ctypes.c_int64 * max(K, 1))(*[c[3] for c in cops])
    n = D * D
    rp = torch.empty(n + 1, dtype=torch.int32, device=dev)
    nnz = ctypes.c_int64(0)
    herm = ctypes.c_double(0.0)
    st = _lib.stream_ptr()
    _lib.call("rs_liouvillian", D, _lib.ptr(hrp), _lib.ptr(hci), _lib.ptr(hv), hnnz, K,
              c_rp, c_ci, c_v, c_nnz, ctypes.byref(herm), _lib.ptr(rp), None, None,
              ctypes.byref(nnz), st)
    if herm.value > _HERM_TOL:
        raise ValueError("Hamiltonian is not Hermitian within 1e-12")
    ci = torch.empty(max(nnz.value, 1), dtype=torch.int32, device=dev)
    v = torch.empty(max(nnz.value, 1), dtype=torch.complex128, device=dev)
    _lib.call("rs_liouvillian", D, _lib.ptr(hrp), _lib.ptr(hci), _lib.ptr(hv), hnnz, K,
              c_rp, c_ci, c_v, c_nnz, None, _lib.ptr(rp), _lib.ptr(ci), _lib.ptr(v),
              ctypes.byref(nnz), st)
    keep = (hrp, hci, hv, cops)  # keep inputs alive until the stream drains
    torch.cuda.current_stream().synchronize()
    del keep
    return DeviceCSR(n, 1, rp, ci[:nnz.value], v[:nnz.value])


def build_liouvillian(H, collapse_ops, device=None):
    """liouville.py:54-77: -i(I(x)H - H^T(x)I) + sum_k [conj(C)(x)C
    - (I(x)C'C + (C'C)^T(x)I)/2], assembled on the GPU."""
    _lib.require_cuda()
    dev = device or torch.device("cuda")
    M = _assemble(H, list(collapse_ops), dev)
    return LiouvillianSystem(M, H.matrix.nrows, "plain")


def concat_systems(mats):
    """Stack single-system DeviceCSRs (equal n) into one block-diagonal batch."""
    n = mats[0].n
    offs, rps, o = [], [], 0
    for m in mats:
        if m.n != n or m.nsys != 1:
            raise ValueError("batch members must be single systems of equal order")
        rps.append(m.row_ptr[:-1] + o)
        o += m.nnz
    rps.append(torch.tensor([o], dtype=torch.int32, device=mats[0].row_ptr.device))
    return DeviceCSR(n, len(mats), torch.cat(rps), torch.cat([m.col_idx for m in mats]),
                     torch.cat([m.values for m in mats]))


def _stack_ops(ops, dev):
    """Block-diagonal batch of D x D operator CSRs (host) on the device:
    absolute row pointers over len(ops)*D rows, local column indices."""
    hs = [as_host_csr(o.matrix) for o in ops]
    D = hs[0].nrows
    nnz = np.fromiter((h.nnz for h in hs), dtype=np.int64, count=len(hs))
    offs = np.concatenate(([0], np.cumsum(nnz)))
    rp = np.empty(len(hs) * D + 1, dtype=np.int32)
    for b, h in enumerate(hs):
        rp[b * D:(b + 1) * D] = h.row_ptr[:-1] + offs[b]
    rp[-1] = offs[-1]
    ci = np.concatenate([h.col_idx for h in hs]).astype(np.int32)
    v = np.ascontiguousarray(np.concatenate([h.values for h in hs]), dtype=np.complex128)
    return (torch.from_numpy(rp).to(dev), torch.from_numpy(ci).to(dev),
            torch.from_numpy(v).to(dev), int(offs[-1]))


def build_liouvillian_batch(models, device=None):
    """Assemble several (H, c_ops) of equal dimension and operator count into
    one block-diagonal plain LiouvillianSystem (the config-4 parameter sweep)
    with ONE launch set for the whole batch (rs_liouvillian_batch): per system
    bit-identical to build_liouvillian."""
    _lib.require_cuda()
    dev = device or torch.device("cuda")
    models = [(H, list(c)) for H, c in models]
    H0, c0 = models[0]
    D, K, B = H0.matrix.nrows, len(c0), len(models)
    for H, c in models:
        if H.matrix.nrows != D or len(c) != K:
            raise ValueError("batch members must share the dimension and operator count")
        for x in c:
            if tuple(x.dims) != tuple(H.dims):
                raise ValueError(f"collapse operator dims {x.dims} do not match H {H.dims}")
    hrp, hci, hv, hnnz = _stack_ops([H for H, _ in models], dev)
    cops = [_stack_ops([c[k] for _, c in models], dev) for k in range(K)]
    PArr = ctypes.c_void_p * max(K, 1)
    c_rp = PArr(*[c[0].data_ptr() for c in cops])
    c_ci = PArr(*[c[1].data_ptr() for c in cops])
    c_v = PArr(*[c[2].data_ptr() for c in cops])
    c_nnz = (ctypes.c_int64 * max(K, 1))(*[c[3] for c in cops])
    n = D * D
    rp = torch.empty(B * n + 1, dtype=torch.int32, device=dev)
    nnz = ctypes.c_int64(0)
    herm = ctypes.c_double(0.0)
    st = _lib.stream_ptr()
    _lib.call("rs_liouvillian_batch", B, D, _lib.ptr(hrp), _lib.ptr(hci), _lib.ptr(hv), hnnz, K,
              c_rp, c_ci, c_v, c_nnz, ctypes.byref(herm), _lib.ptr(rp), None, None,
              ctypes.byref(nnz), st)
    if herm.value > _HERM_TOL:
        raise ValueError("Hamiltonian is not Hermitian within 1e-12")
    ci = torch.empty(max(nnz.value, 1), dtype=torch.int32, device=dev)
    v = torch.empty(max(nnz.value, 1), dtype=torch.complex128, device=dev)
    _lib.call("rs_liouvillian_batch", B, D, _lib.ptr(hrp), _lib.ptr(hci), _lib.ptr(hv), hnnz, K,
              c_rp, c_ci, c_v, c_nnz, None, _lib.ptr(rp), _lib.ptr(ci), _lib.ptr(v),
              ctypes.byref(nnz), st)
    torch.cuda.current_stream().synchronize()  # inputs stay alive until the stream drains
    return LiouvillianSystem(DeviceCSR(n, B, rp, ci[:nnz.value], v[:nnz.value]), D, "plain")


def shift(L, sigma=DEFAULT_SIGMA):
    """liouville.py:80-96: L - sigma I with every diagonal position stored."""
    if L.variant != "plain":
        raise ValueError(f"shift expects the plain variant, got {L.variant!r}")
    if sigma == 0:
        raise ValueError("sigma must be nonzero")
    M = L.matrix
    dev = M.values.device
    rp = torch.empty(M.nsys * M.n + 1, dtype=torch.int32, device=dev)
    nnz = ctypes.c_int64(0)
    st = _lib.stream_ptr()
    _lib.call("rs_shift", M.nsys, M.n, _lib.ptr(M.row_ptr), _lib.ptr(M.col_idx),
              _lib.ptr(M.values), float(sigma), _lib.ptr(rp), None, None, ctypes.byref(nnz), st)
    ci = torch.empty(nnz.value, dtype=torch.int32, device=dev)
    v = torch.empty(nnz.value, dtype=torch.complex128, device=dev)
    _lib.call("rs_shift", M.nsys, M.n, _lib.ptr(M.row_ptr), _lib.ptr(M.col_idx),
              _lib.ptr(M.values), float(sigma), _lib.ptr(rp), _lib.ptr(ci), _lib.ptr(v),
              ctypes.byref(nnz), st)
    return LiouvillianSystem(DeviceCSR(M.n, M.nsys, rp, ci, v), L.hilbert_dim, "shifted",
                             sigma=sigma)


def _weights(L, mode):
    if mode not in ("abs", "signed"):
        raise ValueError(f"unknown weight mode {mode!r}")
    M = L.matrix
    w = torch.empty(M.nsys, dtype=torch.float64, device=M.values.device)
    _lib.call("rs_default_weight", M.nsys, M.n, _lib.ptr(M.row_ptr), _lib.ptr(M.col_idx),
              _lib.ptr(M.values), 0 if mode == "abs" else 1, _lib.ptr(w), _lib.stream_ptr())
    return w


def default_weight(L, mode="abs"):
    """liouville.py:99-111 (one float; an array for a batch)."""
    w = _weights(L, mode).cpu().numpy()
    if not np.all(w > 0):
        raise ValueError("diagonal average vanished; supply w explicitly")
    return float(w[0]) if L.nsys == 1 else w


def build_modified(L, w=None, weight_mode="abs"):
    """liouville.py:114-138: row 0 += w at columns k(D+1); rhs = (w, 0, ...)."""
    if L.variant != "plain":
        raise ValueError(f"build_modified expects the plain variant, got {L.variant!r}")
    M = L.matrix
    dev = M.values.device
    if w is None:
        wt = _weights(L, weight_mode)
        wh = wt.cpu().numpy()
        if not np.all(wh > 0):
            raise ValueError("diagonal average vanished; supply w explicitly")
    else:
        wh = np.broadcast_to(np.asarray(w, dtype=np.float64), (M.nsys,)).copy()
        if not np.all(wh > 0):
            raise ValueError("w must be positive")
        wt = torch.from_numpy(wh).to(dev)
    D = L.hilbert_dim
    rp = torch.empty(M.nsys * M.n + 1, dtype=torch.int32, device=dev)
    nnz = ctypes.c_int64(0)
    st = _lib.stream_ptr()
    _lib.call("rs_trace_modify", M.nsys, M.n, D, _lib.ptr(M.row_ptr), _lib.ptr(M.col_idx),
              _lib.ptr(M.values), _lib.ptr(wt), _lib.ptr(rp), None, None, ctypes.byref(nnz), st)
    ci = torch.empty(nnz.value, dtype=torch.int32, device=dev)
    v = torch.empty(nnz.value, dtype=torch.complex128, device=dev)
    _lib.call("rs_trace_modify", M.nsys, M.n, D, _lib.ptr(M.row_ptr), _lib.ptr(M.col_idx),
              _lib.ptr(M.values), _lib.ptr(wt), _lib.ptr(rp), _lib.ptr(ci), _lib.ptr(v),
              ctypes.byref(nnz), st)
    rhs = torch.zeros(M.nsys, M.n, dtype=torch.complex128, device=dev)
    rhs[:, 0] = wt.to(torch.complex128)
    weight = float(wh[0]) if M.nsys == 1 else wh
    return LiouvillianSystem(DeviceCSR(M.n, M.nsys, rp, ci, v), D, "modified", weight=weight,
                             rhs=rhs.reshape(-1))
