"""Host-side sparse containers and the small operator algebra used to build
model inputs, plus the device CSR type the GPU stages exchange.

`CSRMatrix` mirrors the reference container (pkg/src/rhosolve/sparse.py:30-142:
int64 row pointers / column indices, complex128 values, rows sorted by
strictly increasing column) so the reference's own `QuantumOperator`s and
ours are interchangeable at the drop-in surface.  The host algebra here only
ever touches D x D operators (D <= 1600 in every configuration); everything
n x n (n = D^2) lives on the GPU as `DeviceCSR`.

Semantics that make inputs bit-identical to the reference's:
  * from_coo sums duplicate (row, col) pairs in order of appearance after a
    stable (row, col) sort and prunes exact zeros (sparse.py:77-97);
  * kron/add scale and multiply with numpy array arithmetic
    (sparse.py:202-240);
  * matmul accumulates per output row over the inner index in storage order
    with numpy scalar arithmetic, starting from 0.0 (sparse.py:243-265).
"""

from __future__ import annotations

import numpy as np
import torch

__all__ = ["CSRMatrix", "Permutation", "DeviceCSR", "PinnedBatchCSR", "identity", "kron",
           "transpose", "conjugate", "adjoint", "add", "matmul", "from_host", "pin_batch",
           "as_host_csr", "write_matrix_market", "read_matrix_market"]

_MM_HEADER = "%%MatrixMarket matrix coordinate complex general"


class CSRMatrix:
    """Immutable host CSR matrix (int64 indices, complex128 values)."""

    __slots__ = ("nrows", "ncols", "row_ptr", "col_idx", "values")

    def __init__(self, nrows, ncols, row_ptr, col_idx, values):
        self.nrows = int(nrows)
        self.ncols = int(ncols)
        self.row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
        self.col_idx = np.ascontiguousarray(col_idx, dtype=np.int64)
        self.values = np.ascontiguousarray(values, dtype=np.complex128)
        if len(self.row_ptr) != self.nrows + 1 or self.row_ptr[-1] != len(self.values):
            raise ValueError("inconsistent CSR arrays")

    @property
    def nnz(self):
        return len(self.values)

    @property
    def shape(self):
        return (self.nrows, self.ncols)

    def row_ids(self):
        return np.repeat(np.arange(self.nrows, dtype=np.int64), np.diff(self.row_ptr))

    @classmethod
    def from_coo(cls, nrows, ncols, rows, cols, vals, prune=True):
        rows = np.asarray(rows, dtype=np.int64)
        cols = np.asarray(cols, dtype=np.int64)
        vals = np.asarray(vals, dtype=np.complex128)
        if rows.size:
            perm = np.argsort(rows * max(ncols, 1) + cols, kind="stable")
            rows, cols, vals = rows[perm], cols[perm], vals[perm]
            head = np.empty(rows.size, dtype=bool)
            head[0] = True
            np.not_equal(rows[1:] * max(ncols, 1) + cols[1:],
                         rows[:-1] * max(ncols, 1) + cols[:-1], out=head[1:])
            starts = np.flatnonzero(head)
            vals = np.add.reduceat(vals, starts)
            rows, cols = rows[starts], cols[starts]
            if prune:
                nz = vals != 0
                rows, cols, vals = rows[nz], cols[nz], vals[nz]
        counts = np.bincount(rows, minlength=nrows) if rows.size else np.zeros(nrows, np.int64)
        rp = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        return cls(nrows, ncols, rp, cols, vals)

    def to_dense(self):
        out = np.zeros(self.shape, dtype=np.complex128)
        out[self.row_ids(), self.col_idx] = self.values
        return out

    def to_coo(self):
        return self.row_ids(), self.col_idx.copy(), self.values.copy()

    def diagonal_stored_count(self):
        """How many diagonal positions are explicitly stored (sparse.py:127-131)."""
        return int(np.count_nonzero(self.row_ids() == self.col_idx))

    def __repr__(self):
        return f"CSRMatrix({self.nrows}x{self.ncols}, nnz={self.nnz})"


class Permutation:
    """forward[i] = new position of i; inverse = forward^-1
    (reference sparse.Permutation, sparse.py:145-192)."""

    __slots__ = ("forward", "inverse")

    def __init__(self, forward, inverse=None):
        self.forward = np.ascontiguousarray(forward, dtype=np.int64)
        if inverse is None:
            inverse = np.empty_like(self.forward)
            inverse[self.forward] = np.arange(len(self.forward))
        self.inverse = np.ascontiguousarray(inverse, dtype=np.int64)
        n = len(self.forward)
        if (len(self.inverse) != n
                or not np.array_equal(np.sort(self.forward), np.arange(n))
                or not np.array_equal(self.inverse[self.forward], np.arange(n))):
            raise ValueError("not a bijection with matching inverse")

    @classmethod
    def identity(cls, n):
        idx = np.arange(n, dtype=np.int64)
        return cls(idx, idx)

    @classmethod
    def from_order(cls, order):
        order = np.asarray(order, dtype=np.int64)
        fwd = np.empty_like(order)
        fwd[order] = np.arange(len(order))
        return cls(fwd, order)

    def __len__(self):
        return len(self.forward)

    def is_identity(self):
        return bool(np.array_equal(self.forward, np.arange(len(self.forward))))

    def save(self, path):
        """Newline-delimited forward map (sparse.py:179-183)."""
        with open(path, "w", encoding="ascii") as fh:
            fh.write("\n".join(str(int(i)) for i in self.forward))
            fh.write("\n")

    @classmethod
    def load(cls, path):
        """Inverse of save (sparse.py:185-189)."""
        with open(path, encoding="ascii") as fh:
            vals = [int(line) for line in fh if line.strip()]
        return cls(np.array(vals, dtype=np.int64))

    def __repr__(self):
        return f"Permutation(n={len(self.forward)})"


def identity(n):
    idx = np.arange(n, dtype=np.int64)
    return CSRMatrix(n, n, np.arange(n + 1), idx, np.ones(n, dtype=np.complex128))


def kron(a, b):
    """((i*b.nrows + k), (j*b.ncols + l)) = a[i,j] * b[k,l]."""
    ar, ac, av = a.to_coo()
    br, bc, bv = b.to_coo()
    rows = (ar[:, None] * b.nrows + br[None, :]).ravel()
    cols = (ac[:, None] * b.ncols + bc[None, :]).ravel()
    vals = (av[:, None] * bv[None, :]).ravel()
    return CSRMatrix.from_coo(a.nrows * b.nrows, a.ncols * b.ncols, rows, cols, vals,
                              prune=False)


def transpose(a):
    r, c, v = a.to_coo()
    return CSRMatrix.from_coo(a.ncols, a.nrows, c, r, v, prune=False)


def conjugate(a):
    return CSRMatrix(a.nrows, a.ncols, a.row_ptr, a.col_idx, np.conj(a.values))


def adjoint(a):
    return conjugate(transpose(a))


def add(a, b, alpha=1.0, beta=1.0):
    if a.shape != b.shape:
        raise ValueError(f"shape mismatch: {a.shape} vs {b.shape}")
    ar, ac, av = a.to_coo()
    br, bc, bv = b.to_coo()
    return CSRMatrix.from_coo(a.nrows, a.ncols, np.concatenate([ar, br]),
                              np.concatenate([ac, bc]),
                              np.concatenate([alpha * av, beta * bv]))


def matmul(a, b):
    """Row-merge product with scalar accumulation in storage order."""
    if a.ncols != b.nrows:
        raise ValueError(f"shape mismatch: {a.shape} @ {b.shape}")
    rows, cols, vals = [], [], []
    bp, bi, bv = b.row_ptr, b.col_idx, b.values
    for i in range(a.nrows):
        acc = {}
        for p in range(a.row_ptr[i], a.row_ptr[i + 1]):
            j = a.col_idx[p]
            s = a.values[p]
            for t in range(bp[j], bp[j + 1]):
                key = int(bi[t])
                acc[key] = acc.get(key, 0.0) + s * bv[t]
        for key, val in acc.items():
            rows.append(i)
            cols.append(key)
            vals.append(val)
    return CSRMatrix.from_coo(a.nrows, b.ncols, rows, cols, vals)


def as_host_csr(m):
    """Accept our CSRMatrix, a single-system DeviceCSR, a system object with
    .matrix, or the reference SparseComplexMatrix (duck-typed)."""
    if isinstance(m, CSRMatrix):
        return m
    if not hasattr(m, "row_ptr") and hasattr(m, "matrix"):
        m = m.matrix
    if isinstance(m, DeviceCSR):
        return m.to_host()
    return CSRMatrix(m.nrows, m.ncols, m.row_ptr, m.col_idx, m.values)


class DeviceCSR:
    """Block-diagonal batch of `nsys` n-by-n CSR matrices on the GPU:
    int32 row_ptr over nsys*n rows (absolute positions), int32 local column
    indices, complex128 values (the C-ABI layout of include/rhosolve_b200.h)."""

    __slots__ = ("n", "nsys", "row_ptr", "col_idx", "values")

    def __init__(self, n, nsys, row_ptr, col_idx, values):
        self.n = int(n)
        self.nsys = int(nsys)
        self.row_ptr = row_ptr
        self.col_idx = col_idx
        self.values = values

    @property
    def nnz(self):
        return int(self.values.numel())

    @property
    def nrows(self):
        return self.n

    @property
    def ncols(self):
        return self.n

    @property
    def shape(self):
        return (self.n, self.n)

    def system(self, b):
        """Host CSRMatrix copy of system b."""
        rp = self.row_ptr.cpu().numpy().astype(np.int64)
        lo, hi = rp[b * self.n], rp[(b + 1) * self.n]
        return CSRMatrix(self.n, self.n, rp[b * self.n:(b + 1) * self.n + 1] - lo,
                         self.col_idx[lo:hi].cpu().numpy(), self.values[lo:hi].cpu().numpy())

    def to_host(self):
        if self.nsys != 1:
            raise ValueError("to_host() on a batch; use system(b)")
        return self.system(0)

    def __repr__(self):
        return f"DeviceCSR(n={self.n}, nsys={self.nsys}, nnz={self.nnz})"


class PinnedBatchCSR:
    """A block-diagonal batch of equal-order CSR matrices staged in pinned
    (page-locked) host memory in the DeviceCSR layout (int32 row_ptr over
    nsys*n rows, int32 local column indices, complex128 values), so that
    `from_host` moves it with three asynchronous DMA copies."""

    __slots__ = ("n", "nsys", "row_ptr", "col_idx", "values")

    def __init__(self, n, nsys, row_ptr, col_idx, values):
        self.n, self.nsys = int(n), int(nsys)
        self.row_ptr, self.col_idx, self.values = row_ptr, col_idx, values

    @property
    def nnz(self):
        return int(self.values.numel())

    @property
    def nbytes(self):
        return 4 * self.row_ptr.numel() + 4 * self.col_idx.numel() + 16 * self.values.numel()


def _pack(mats):
    mats = [as_host_csr(m) for m in mats]
    n = mats[0].nrows
    if any(m.nrows != n or m.ncols != n for m in mats):
        raise ValueError("batch members must be square of equal order")
    offs = np.cumsum([0] + [m.nnz for m in mats])
    if offs[-1] >= 2 ** 31:
        raise ValueError("nnz exceeds int32 indexing")
    return mats, n, offs


def pin_batch(mats):
    """Pack host CSRs (one, or a list of equal order) into a PinnedBatchCSR."""
    if not isinstance(mats, (list, tuple)):
        mats = [mats]
    mats, n, offs = _pack(mats)
    B, nnz = len(mats), int(offs[-1])
    rp = torch.empty(B * n + 1, dtype=torch.int32, pin_memory=True)
    ci = torch.empty(nnz, dtype=torch.int32, pin_memory=True)
    v = torch.empty(nnz, dtype=torch.complex128, pin_memory=True)
    rpn, cin, vn = rp.numpy(), ci.numpy(), v.numpy()
    for b, (m, o) in enumerate(zip(mats, offs[:-1])):
        rpn[b * n:(b + 1) * n] = m.row_ptr[:-1] + o
        cin[o:o + m.nnz] = m.col_idx
        vn[o:o + m.nnz] = m.values
    rpn[B * n] = nnz
    return PinnedBatchCSR(n, B, rp, ci, v)


def from_host(mats, device=None, values_stream=None):
    """Upload one CSR, a list of equal-order CSRs (as a batch), or a
    PinnedBatchCSR (asynchronous copies on the current stream) to the GPU.
    values_stream (pinned batches): the values travel on that stream instead,
    so structure-only work (RCM) can start as soon as row_ptr / col_idx have
    landed; the caller makes its stream wait for values_stream before any
    kernel reads the values."""
    dev = device or torch.device("cuda")
    if isinstance(mats, PinnedBatchCSR):
        rp = mats.row_ptr.to(dev, non_blocking=True)
        ci = mats.col_idx.to(dev, non_blocking=True)
        if values_stream is None:
            v = mats.values.to(dev, non_blocking=True)
        else:
            main = torch.cuda.current_stream(dev)
            values_stream.wait_stream(main)
            with torch.cuda.stream(values_stream):
                v = mats.values.to(dev, non_blocking=True)
            v.record_stream(main)
        return DeviceCSR(mats.n, mats.nsys, rp, ci, v)
    if not isinstance(mats, (list, tuple)):
        mats = [mats]
    mats, n, offs = _pack(mats)
    rp = np.concatenate([m.row_ptr[:-1] + o for m, o in zip(mats, offs[:-1])] + [[offs[-1]]])
    return DeviceCSR(
        n, len(mats),
        torch.from_numpy(rp.astype(np.int32)).to(dev),
        torch.from_numpy(np.concatenate([m.col_idx for m in mats]).astype(np.int32)).to(dev),
        torch.from_numpy(np.concatenate([m.values for m in mats])).to(dev))


def write_matrix_market(a, path, comment=None):
    """Matrix Market coordinate complex general, 1-based indices, values with
    17 significant digits -- the reference writer's bytes (sparse.py:302-312).
    Accepts a host CSRMatrix, a single-system DeviceCSR or any object with
    nrows/ncols/row_ptr/col_idx/values."""
    a = as_host_csr(a)
    rows, cols, vals = a.to_coo()
    lines = [_MM_HEADER]
    if comment:
        lines += [f"% {line}" for line in comment.splitlines()]
    lines.append(f"{a.nrows} {a.ncols} {a.nnz}")
    re, im = vals.real.tolist(), vals.imag.tolist()
    lines += [f"{r + 1} {c + 1} {x:.17g} {y:.17g}"
              for r, c, x, y in zip(rows.tolist(), cols.tolist(), re, im)]
    with open(path, "w", encoding="ascii") as fh:
        fh.write("\n".join(lines) + "\n")


def read_matrix_market(path):
    """Reader for coordinate general complex / real / integer Matrix Market
    files (sparse.py:315-351): duplicates summed, nothing pruned."""
    with open(path, encoding="ascii") as fh:
        header = fh.readline().strip()
        fields = header.lower().split()
        if (len(fields) < 5 or fields[0] != "%%matrixmarket"
                or fields[1] != "matrix" or fields[2] != "coordinate"):
            raise ValueError(f"unsupported Matrix Market header: {header}")
        kind, symmetry = fields[3], fields[4]
        if symmetry != "general":
            raise ValueError(f"unsupported symmetry: {symmetry}")
        if kind not in ("complex", "real", "integer"):
            raise ValueError(f"unsupported field type: {kind}")
        line = fh.readline()
        while line.startswith("%") or not line.strip():
            line = fh.readline()
        nrows, ncols, nnz = (int(t) for t in line.split())
        rows = np.empty(nnz, dtype=np.int64)
        cols = np.empty(nnz, dtype=np.int64)
        vals = np.empty(nnz, dtype=np.complex128)
        got = 0
        for line in fh:
            line = line.strip()
            if not line or line.startswith("%"):
                continue
            parts = line.split()
            if got >= nnz:
                got += 1
                break
            rows[got] = int(parts[0]) - 1
            cols[got] = int(parts[1]) - 1
            vals[got] = (complex(float(parts[2]), float(parts[3])) if kind == "complex"
                         else float(parts[2]))
            got += 1
        if got != nnz:
            raise ValueError(f"expected {nnz} entries, found {got}")
    return CSRMatrix.from_coo(nrows, ncols, rows, cols, vals, prune=False)
