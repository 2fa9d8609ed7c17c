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


def _from_sorted_keys(nrows, ncols, keys, vals):
    """CSR from flat keys (row * ncols + col) that are already unique and
    ascending."""
    keys = np.asarray(keys, dtype=np.int64)
    width = max(ncols, 1)
    rp = np.zeros(nrows + 1, dtype=np.int64)
    np.cumsum(np.bincount(keys // width, minlength=nrows), out=rp[1:])
    return CSRMatrix(nrows, ncols, rp, keys % width, vals)


def _flat_keys(a):
    return a.row_ids() * max(a.ncols, 1) + a.col_idx


def identity(n):
    """The n x n identity."""
    return _from_sorted_keys(n, n, np.arange(n, dtype=np.int64) * (max(n, 1) + 1),
                             np.ones(n, dtype=np.complex128))


def kron(a, b):
    """Kronecker product: entry (i*b.nrows + k, j*b.ncols + l) = a[i,j] * b[k,l]
    (sparse.py:202-213).  The value products are one outer ufunc call, the
    arithmetic the reference's broadcast product performs."""
    rows = np.add.outer(a.row_ids() * b.nrows, b.row_ids()).ravel()
    cols = np.add.outer(a.col_idx * b.ncols, b.col_idx).ravel()
    vals = np.multiply.outer(a.values, b.values).ravel()
    # a's entries are (row, col)-sorted and so are b's, but the combined keys
    # interleave: let from_coo order them (no duplicates can arise)
    return CSRMatrix.from_coo(a.nrows * b.nrows, a.ncols * b.ncols, rows, cols, vals,
                              prune=False)


def transpose(a):
    """a^T: a stable sort of the entries by column keeps rows ascending inside
    every new row, which is exactly the (row, col) order CSR needs."""
    order = np.argsort(a.col_idx, kind="stable")
    rp = np.zeros(a.ncols + 1, dtype=np.int64)
    np.cumsum(np.bincount(a.col_idx, minlength=a.ncols), out=rp[1:])
    return CSRMatrix(a.ncols, a.nrows, rp, a.row_ids()[order], a.values[order])


def conjugate(a):
    return CSRMatrix(a.nrows, a.ncols, a.row_ptr, a.col_idx, a.values.conj())


def adjoint(a):
    return transpose(conjugate(a))


def add(a, b, alpha=1.0, beta=1.0):
    """alpha*a + beta*b with exact zeros dropped (sparse.py:231-240): positions
    in both operands hold (alpha*a) + (beta*b), the others the scaled entry
    itself."""
    if a.shape != b.shape:
        raise ValueError(f"shape mismatch: {a.shape} vs {b.shape}")
    ka, kb = _flat_keys(a), _flat_keys(b)
    va, vb = alpha * a.values, beta * b.values
    keys = np.union1d(ka, kb)
    out = np.empty(len(keys), dtype=np.complex128)
    ia, ib = np.searchsorted(keys, ka), np.searchsorted(keys, kb)
    out[ia] = va
    shared = np.isin(kb, ka, assume_unique=True)
    out[ib[~shared]] = vb[~shared]
    out[ib[shared]] = out[ib[shared]] + vb[shared]
    keep = out != 0
    return _from_sorted_keys(a.nrows, a.ncols, keys[keep], out[keep])


def matmul(a, b):
    """a @ b (sparse.py:243-265).  Every output entry accumulates its products
    from 0 in the order (entry of a's row, entry of b's row), each product in
    the two-rounding complex form of a numpy scalar multiply; exact zeros are
    dropped.  Vectorised: all products are generated in that order and
    np.add.at folds them in sequence."""
    if a.ncols != b.nrows:
        raise ValueError(f"shape mismatch: {a.shape} @ {b.shape}")
    if a.nnz == 0 or b.nnz == 0:
        return _from_sorted_keys(a.nrows, b.ncols, np.empty(0, np.int64),
                                 np.empty(0, np.complex128))
    first = b.row_ptr[a.col_idx]
    count = b.row_ptr[a.col_idx + 1] - first
    src_a = np.repeat(np.arange(a.nnz, dtype=np.int64), count)
    # position inside b: first[src] + (running index within the group)
    start_of_group = np.repeat(np.cumsum(count) - count, count)
    src_b = np.repeat(first, count) + (np.arange(len(src_a), dtype=np.int64) - start_of_group)
    x, y = a.values[src_a], b.values[src_b]
    prod = np.empty(len(src_a), dtype=np.complex128)
    prod.real = x.real * y.real - x.imag * y.imag
    prod.imag = x.real * y.imag + x.imag * y.real
    keys = a.row_ids()[src_a] * max(b.ncols, 1) + b.col_idx[src_b]
    uniq, slot = np.unique(keys, return_inverse=True)
    acc = np.zeros(len(uniq), dtype=np.complex128)
    np.add.at(acc, slot, prod)
    keep = acc != 0
    return _from_sorted_keys(a.nrows, b.ncols, uniq[keep], acc[keep])


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


def _mm_tokens(handle):
    """Whitespace-separated fields of the non-comment, non-blank lines."""
    for raw in handle:
        text = raw.strip()
        if text and not text.startswith("%"):
            yield text.split()


def read_matrix_market(path):
    """Matrix Market coordinate/general reader for complex, real and integer
    fields (the files sparse.py:315-351 accepts): 1-based indices, duplicate
    positions summed, explicit zeros kept."""
    with open(path, encoding="ascii") as handle:
        banner = handle.readline().split()
        tag = [t.lower() for t in banner]
        if len(tag) < 5 or tag[:3] != ["%%matrixmarket", "matrix", "coordinate"]:
            raise ValueError(f"unsupported Matrix Market header: {' '.join(banner)}")
        field, symmetry = tag[3], tag[4]
        if symmetry != "general":
            raise ValueError(f"unsupported symmetry: {symmetry}")
        if field not in ("complex", "real", "integer"):
            raise ValueError(f"unsupported field type: {field}")
        body = _mm_tokens(handle)
        nrows, ncols, nnz = (int(t) for t in next(body))
        entries = list(body)
    if len(entries) != nnz:
        raise ValueError(f"expected {nnz} entries, found {len(entries)}")
    index = np.array([[int(e[0]), int(e[1])] for e in entries], dtype=np.int64).reshape(-1, 2)
    vals = np.empty(nnz, dtype=np.complex128)
    vals.real = [float(e[2]) for e in entries]
    vals.imag = [float(e[3]) for e in entries] if field == "complex" else 0.0
    return CSRMatrix.from_coo(nrows, ncols, index[:, 0] - 1, index[:, 1] - 1, vals, prune=False)
