"""rhosolve-b200 ORACLE -- test infrastructure, not product code.

CPU restatement of the reference steady-state hot path, used only as the
checker by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg.
The product (paper_1504_06768_b200/) never imports it.

Kernels come from oracle/rs_oracle.c (plain C, bit-faithful to the Cython
kernels); the orchestration below restates the reference drivers with numpy:
  assembly        liouville.py:54-138, sparse.py:77-97,202-265
  permute         sparse.py:276-282
  _factor / lu / ilutp / solve_lu / condest   factor.py:70-157
  gmres / bicgstab                            krylov.py:67-291
  _postprocess / solve_direct / solve_iterative / inverse_power
                                              steady.py:62-260
Pinned against the reference: tests/golden/*.npz (made by
tests/golden/make_golden.py from the reference itself) and, where the
reference build exists (oracle/_ref, git-ignored), directly against it.
"""

from __future__ import annotations

import ctypes
import math
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "_build", "librs_oracle.so")

_c = None


def _lib():
    global _c
    if _c is None:
        if not os.path.exists(_LIB):
            import subprocess
            subprocess.check_call(["make", "-s", "-C", _HERE])
        _c = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        I = ctypes.c_int64
        _c.orc_csr_matvec.argtypes = [I, P, P, P, P, P]
        _c.orc_lower_solve.argtypes = [I, P, P, P, P]
        _c.orc_upper_solve.argtypes = [I, P, P, P, P]
        _c.orc_factorize.argtypes = [I, P, P, P, P, ctypes.c_double, I, P, P]
        _c.orc_factorize.restype = ctypes.c_int
        _c.orc_factorize_opts.argtypes = [I, P, P, P, P, ctypes.c_double, I, P,
                                          ctypes.c_double, ctypes.c_int, P, P]
        _c.orc_factorize_opts.restype = ctypes.c_int
        _c.orc_free_factors.argtypes = [P]
        _c.orc_rcm.argtypes = [I, P, P, P]
        _c.orc_rcm.restype = ctypes.c_int
    return _c


class _Factors(ctypes.Structure):
    _fields_ = [("Lp", ctypes.c_void_p), ("Li", ctypes.c_void_p), ("Up", ctypes.c_void_p),
                ("Ui", ctypes.c_void_p), ("pinv", ctypes.c_void_p), ("Lx", ctypes.c_void_p),
                ("Ux", ctypes.c_void_p), ("lnnz", ctypes.c_int64), ("unnz", ctypes.c_int64),
                ("fail_col", ctypes.c_int64)]


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _c128(a):
    return np.ascontiguousarray(a, dtype=np.complex128)


# ---------------------------------------------------------------- CSR ------
class CSR:
    """Minimal CSR (int64 / complex128), same layout as the reference."""

    __slots__ = ("n", "m", "rp", "ci", "v")

    def __init__(self, n, m, rp, ci, v):
        self.n, self.m = int(n), int(m)
        self.rp, self.ci, self.v = _i64(rp), _i64(ci), _c128(v)

    @property
    def nnz(self):
        return len(self.v)

    def rows(self):
        return np.repeat(np.arange(self.n, dtype=np.int64), np.diff(self.rp))

    def dense(self):
        d = np.zeros((self.n, self.m), dtype=np.complex128)
        d[self.rows(), self.ci] = self.v
        return d


def csr_of(m):
    """From any object with nrows/ncols/row_ptr/col_idx/values."""
    return CSR(m.nrows, m.ncols, m.row_ptr, m.col_idx, m.values)


def coo_to_csr(n, m, r, c, v, prune):
    r, c, v = _i64(r), _i64(c), _c128(v)
    if r.size:
        key = r * max(m, 1) + c
        o = np.argsort(key, kind="stable")
        r, c, v, key = r[o], c[o], v[o], key[o]
        first = np.r_[True, key[1:] != key[:-1]]
        idx = np.flatnonzero(first)
        v = np.add.reduceat(v, idx)
        r, c = r[idx], c[idx]
        if prune:
            keep = v != 0
            r, c, v = r[keep], c[keep], v[keep]
    rp = np.zeros(n + 1, dtype=np.int64)
    if r.size:
        rp[1:] = np.cumsum(np.bincount(r, minlength=n))
    return CSR(n, m, rp, c, v)


def kron(a, b):
    ar, br = a.rows(), b.rows()
    rr = (ar[:, None] * b.n + br[None, :]).ravel()
    cc = (a.ci[:, None] * b.m + b.ci[None, :]).ravel()
    vv = (a.v[:, None] * b.v[None, :]).ravel()
    return coo_to_csr(a.n * b.n, a.m * b.m, rr, cc, vv, prune=False)


def transpose(a):
    return coo_to_csr(a.m, a.n, a.ci, a.rows(), a.v, prune=False)


def add(a, b, alpha=1.0, beta=1.0):
    return coo_to_csr(a.n, a.m, np.r_[a.rows(), b.rows()], np.r_[a.ci, b.ci],
                      np.r_[alpha * a.v, beta * b.v], prune=True)


def adjoint_times_self(c):
    """C^dag C with the reference's per-row scalar accumulation."""
    ct = transpose(c)
    rows, cols, vals = [], [], []
    for i in range(ct.n):
        acc = {}
        for p in range(ct.rp[i], ct.rp[i + 1]):
            j, s = ct.ci[p], np.conj(ct.v[p])
            for t in range(c.rp[j], c.rp[j + 1]):
                k = int(c.ci[t])
                acc[k] = acc.get(k, 0.0) + s * c.v[t]
        for k, val in acc.items():
            rows.append(i)
            cols.append(k)
            vals.append(val)
    return coo_to_csr(c.m, c.m, rows, cols, vals, prune=True)


def identity(n):
    return CSR(n, n, np.arange(n + 1), np.arange(n), np.ones(n))


def build_liouvillian(H, c_ops):
    """liouville.py:54-77 as a chain of sorted merges."""
    h = csr_of(H)
    D = h.n
    eye = identity(D)
    L = add(kron(eye, h), kron(transpose(h), eye), -1j, 1j)
    for op in c_ops:
        c = csr_of(op)
        cdc = adjoint_times_self(c)
        cbar = CSR(c.n, c.m, c.rp, c.ci, np.conj(c.v))
        L = add(L, kron(cbar, c))
        L = add(L, kron(eye, cdc), 1.0, -0.5)
        L = add(L, kron(transpose(cdc), eye), 1.0, -0.5)
    return L


def shift(L, sigma=1e-15):
    n = L.n
    d = np.arange(n)
    return coo_to_csr(n, n, np.r_[L.rows(), d], np.r_[L.ci, d],
                      np.r_[L.v, np.full(n, -sigma, dtype=np.complex128)], prune=False)


def default_weight(L, mode="abs"):
    d = np.zeros(L.n, dtype=np.complex128)
    r = L.rows()
    on = r == L.ci
    d[r[on]] = L.v[on]
    w = float(np.mean(np.abs(d))) if mode == "abs" else float(abs(np.mean(d)))
    if not w > 0:
        raise ValueError("diagonal average vanished")
    return w


def build_modified(L, D, w=None):
    if w is None:
        w = default_weight(L)
    n = L.n
    tc = np.arange(D, dtype=np.int64) * (D + 1)
    m = coo_to_csr(n, n, np.r_[L.rows(), np.zeros(D, np.int64)], np.r_[L.ci, tc],
                   np.r_[L.v, np.full(D, w, dtype=np.complex128)], prune=False)
    rhs = np.zeros(n, dtype=np.complex128)
    rhs[0] = w
    return m, rhs, w


# ------------------------------------------------------------- kernels -----
def csr_matvec(A, x):
    x = _c128(x)
    y = np.empty(A.n, dtype=np.complex128)
    _lib().orc_csr_matvec(A.n, _p(A.rp), _p(A.ci), _p(A.v), _p(x), _p(y))
    return y


def rcm_order(A):
    """Cuthill-McKee order (not reversed), ordering.py:82-118."""
    order = np.empty(A.n, dtype=np.int64)
    if _lib().orc_rcm(A.n, _p(A.rp), _p(A.ci), _p(order)) != 0:
        raise MemoryError
    return order


def rcm(A):
    """(forward, inverse) of the reversed CM order (Permutation.from_order)."""
    inv = rcm_order(A)[::-1].copy()
    fwd = np.empty_like(inv)
    fwd[inv] = np.arange(len(inv))
    return fwd, inv


def permute(A, fwd):
    return coo_to_csr(A.n, A.m, fwd[A.rows()], fwd[A.ci], A.v, prune=False)


class Breakdown(Exception):
    def __init__(self, step, incomplete):
        super().__init__(f"zero pivot at elimination step {step}")
        self.step = step
        self.incomplete = incomplete


class Factors:
    __slots__ = ("n", "Lp", "Li", "Lx", "Up", "Ui", "Ux", "pinv", "fill_factor", "nfloor")

    def solve(self, b):
        """factor.solve_lu with identity column permutation."""
        y = np.empty(self.n, dtype=np.complex128)
        y[self.pinv] = b
        lib = _lib()
        lib.orc_lower_solve(self.n, _p(self.Lp), _p(self.Li), _p(self.Lx), _p(y))
        lib.orc_upper_solve(self.n, _p(self.Up), _p(self.Ui), _p(self.Ux), _p(y))
        return y


def factorize_raw(A, drop_tol, fill_limit, q=None, pivot_floor=0.0, early_drop=False):
    """factor._factor (factor.py:70-112) -> Factors, or raises Breakdown.
    q: elimination column order (col_perm.inverse, factor.py:78).
    pivot_floor > 0: the opt-in zero-pivot substitution (not in the reference;
    see rs_oracle.c orc_factorize_opts); Factors.nfloor counts them.
    early_drop: the opt-in Saad-ILUT rule (drop before eliminating)."""
    n = A.n
    at = transpose(A)
    incomplete = drop_tol > 0.0 or not math.isinf(fill_limit)
    rn = None
    if drop_tol > 0.0:
        rn = np.zeros(n)
        np.maximum.at(rn, A.rows(), np.abs(A.v.real) + np.abs(A.v.imag))
    cap = -1 if math.isinf(fill_limit) else int(math.ceil(fill_limit * A.nnz / n))
    out = _Factors()
    qa = None if q is None else _i64(q)
    nfloor = ctypes.c_int64(0)
    if _lib().orc_factorize_opts(n, _p(at.rp), _p(at.ci), _p(at.v), _p(qa), float(drop_tol),
                                 cap, _p(rn), float(pivot_floor), int(bool(early_drop)),
                                 ctypes.byref(nfloor), ctypes.byref(out)) != 0:
        raise MemoryError
    try:
        if out.fail_col >= 0:
            raise Breakdown(int(out.fail_col), incomplete)

        def arr(ptr, cnt, dt):
            buf = (ctypes.c_char * (cnt * np.dtype(dt).itemsize)).from_address(ptr)
            return np.frombuffer(buf, dtype=dt).copy()

        f = Factors()
        f.n = n
        f.Lp = arr(out.Lp, n + 1, np.int64)
        f.Up = arr(out.Up, n + 1, np.int64)
        f.Li = arr(out.Li, out.lnnz, np.int64)
        f.Lx = arr(out.Lx, out.lnnz, np.complex128)
        f.Ui = arr(out.Ui, out.unnz, np.int64)
        f.Ux = arr(out.Ux, out.unnz, np.complex128)
        f.pinv = arr(out.pinv, n, np.int64)
        f.fill_factor = (out.lnnz + out.unnz) / A.nnz
        f.nfloor = int(nfloor.value)
        return f
    finally:
        _lib().orc_free_factors(ctypes.byref(out))


def condest(f):
    return float(np.max(np.abs(f.solve(np.ones(f.n, dtype=np.complex128)))))


# -------------------------------------------------------------- Krylov -----
def bicgstab(A, b, M, tol, max_iter):
    """krylov.py:181-291 -> (x, iterations, converged, breakdown)."""
    ps = (lambda v: M.solve(v)) if M is not None else (lambda v: v)
    n = A.n
    bnorm = np.linalg.norm(b)
    if bnorm == 0.0:
        return np.zeros(n, complex), 0, True, False
    pb = ps(b)
    pbn = np.linalg.norm(pb)
    if pbn == 0.0 or not np.isfinite(pbn):
        return np.zeros(n, complex), 0, False, True
    x = np.zeros(n, complex)
    r = pb.copy()
    rh = r.copy()
    rhn = np.linalg.norm(rh)
    rho_old = alpha = omega = 1.0 + 0.0j
    v = np.zeros(n, complex)
    p = np.zeros(n, complex)
    target, prev, it = tol * pbn, np.inf, 0
    conv = brk = False
    while it < max_iter:
        rn = np.linalg.norm(r)
        if rn <= target:
            tr = np.linalg.norm(b - csr_matvec(A, x))
            if tr <= tol * bnorm:
                conv = True
                break
            if tr >= 0.5 * prev:
                break
            prev, target = tr, target * 0.1
        rho = np.vdot(rh, r)
        if abs(rho) < 1e-30 or abs(rho) < 1e-16 * rhn * rn:
            brk = True
            break
        if it == 0:
            p[:] = r
        else:
            p = r + (rho / rho_old) * (alpha / omega) * (p - omega * v)
        v = ps(csr_matvec(A, p))
        den = np.vdot(rh, v)
        if den == 0.0:
            brk = True
            break
        alpha = rho / den
        s = r - alpha * v
        it += 1
        if np.linalg.norm(s) <= target:
            x = x + alpha * p
            tr = np.linalg.norm(b - csr_matvec(A, x))
            if tr <= tol * bnorm:
                conv = True
                break
            if tr >= 0.5 * prev:
                break
            prev, target = tr, target * 0.1
            r = s
            rh = r.copy()
            rhn = np.linalg.norm(rh)
            rho_old = alpha = omega = 1.0 + 0.0j
            v[:] = 0.0
            p[:] = 0.0
            continue
        t = ps(csr_matvec(A, s))
        tt = np.vdot(t, t)
        if tt == 0.0:
            brk = True
            break
        omega = np.vdot(t, s) / tt
        x = x + alpha * p + omega * s
        r = s - omega * t
        rho_old = rho
        if omega == 0.0:
            brk = True
            break
    return x, it, conv, brk


def gmres(A, b, M, tol, max_iter, m):
    """krylov.py:67-178 -> (x, iterations, converged, breakdown)."""
    ps = (lambda v: M.solve(v)) if M is not None else (lambda v: v)
    n = A.n
    bnorm = np.linalg.norm(b)
    if bnorm == 0.0:
        return np.zeros(n, complex), 0, True, False
    pb = ps(b)
    pbn = np.linalg.norm(pb)
    if pbn == 0.0 or not np.isfinite(pbn):
        return np.zeros(n, complex), 0, False, True
    x = np.zeros(n, complex)
    target, total, prev = tol * pbn, 0, np.inf
    conv = brk = inv = False
    V = np.empty((m + 1, n), complex)
    H = np.zeros((m + 1, m), complex)
    cs = np.zeros(m)
    sn = np.zeros(m, complex)
    g = np.zeros(m + 1, complex)
    while total < max_iter and not conv and not inv:
        r = pb - ps(csr_matvec(A, x)) if total else pb.copy()
        beta = np.linalg.norm(r)
        hit = beta <= target
        if not hit:
            V[0] = r / beta
            g[:] = 0.0
            g[0] = beta
            H[:, :] = 0.0
            j, res = 0, beta
            while j < m and total < max_iter:
                w = ps(csr_matvec(A, V[j]))
                total += 1
                for i in range(j + 1):
                    H[i, j] = np.vdot(V[i], w)
                    w -= H[i, j] * V[i]
                hn = np.linalg.norm(w)
                if hn > 0.0:
                    V[j + 1] = w / hn
                for i in range(j):
                    t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                    H[i + 1, j] = -np.conj(sn[i]) * H[i, j] + cs[i] * H[i + 1, j]
                    H[i, j] = t
                a = H[j, j]
                den = np.hypot(abs(a), hn)
                if den == 0.0:
                    cs[j], sn[j] = 1.0, 0.0
                elif a == 0.0:
                    cs[j], sn[j] = 0.0, 1.0
                else:
                    cs[j] = abs(a) / den
                    sn[j] = (a / abs(a)) * (hn / den)
                H[j, j] = cs[j] * a + sn[j] * hn
                g[j + 1] = -np.conj(sn[j]) * g[j]
                g[j] = cs[j] * g[j]
                res = abs(g[j + 1])
                j += 1
                if hn == 0.0:
                    inv = True
                    break
                if res <= target:
                    break
            if np.any(np.diagonal(H)[:j] == 0.0):
                brk = True
                break
            y = np.zeros(j, complex)
            for i in range(j - 1, -1, -1):
                y[i] = (g[i] - H[i, i + 1:j] @ y[i + 1:j]) / H[i, i]
            x = x + y @ V[:j]
            hit = res <= target or inv
        if hit:
            tr = np.linalg.norm(b - csr_matvec(A, x))
            if tr <= tol * bnorm:
                conv = True
            elif inv or tr >= 0.5 * prev:
                break
            else:
                prev, target = tr, target * 0.1
    return x, total, conv, brk


# ------------------------------------------------------------- drivers -----
def postprocess(x, D, plain):
    rho = _c128(x).reshape(D, D).T.copy()
    rho = 0.5 * (rho + rho.conj().T)
    tr = np.trace(rho)
    if tr != 0:
        rho = rho / tr
    return rho, float(np.linalg.norm(csr_matvec(plain, rho.T.reshape(-1))))


def start_vector(n, seed):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    return x / np.linalg.norm(x)


def inverse_power(L, D, sigma=1e-15, tol=1e-14, inner="direct", ordering="rcm",
                  solver="gmres", d=1e-4, p=300.0, restart_m=20, max_iter=1000, seed=12345,
                  max_outer=50):
    """steady.py:177-260.  Returns dict(rho, residual, outer, inner, fill, condest)."""
    m = shift(L, sigma)
    fwd = None
    if ordering == "rcm":
        fwd, _ = rcm(m)
        m = permute(m, fwd)
        plain = permute(L, fwd)
    else:
        plain = L
    if inner == "direct":
        f = factorize_raw(m, 0.0, math.inf)
        cond = None
    else:
        f = factorize_raw(m, d, float(p))
        cond = condest(f)
    x = start_vector(m.n, seed)
    outer, inner_its, conv = 0, [], False
    while outer < max_outer:
        if inner == "direct":
            y = f.solve(x)
        else:
            run = gmres if solver == "gmres" else bicgstab
            args = (restart_m,) if solver == "gmres" else ()
            y, its, _, brk = run(m, x, f, tol / 10, max_iter, *args)
            inner_its.append(its)
            if brk or not np.all(np.isfinite(y)) or np.linalg.norm(y) == 0.0:
                raise RuntimeError("InnerSolverError")
        ny = np.linalg.norm(y)
        y = y / ny
        outer += 1
        ov = np.vdot(y, x)
        aligned = y * (ov / abs(ov)) if ov != 0 else y
        diff = np.linalg.norm(aligned - x)
        rinf = float(np.max(np.abs(csr_matvec(plain, y))))
        x = y
        if diff <= tol or rinf <= tol:
            conv = True
            break
    if not conv:
        raise RuntimeError("PowerIterationError")
    if fwd is not None:
        x = x[fwd]
    rho, res = postprocess(x, D, L)
    return dict(rho=rho, residual=res, outer=outer, inner=inner_its,
                fill=f.fill_factor, condest=cond, perm=fwd)


def solve_linear(L, D, method="bicgstab", ordering="rcm", d=1e-4, p=300.0, tol=1e-14,
                 restart_m=20, max_iter=1000, w=None):
    """steady.solve_iterative / solve_direct (method="direct")."""
    m, rhs, w = build_modified(L, D, w)
    fwd = None
    if ordering == "rcm":
        fwd, _ = rcm(m)
        m = permute(m, fwd)
        prhs = np.empty_like(rhs)
        prhs[fwd] = rhs
        rhs = prhs
    if method == "direct":
        f = factorize_raw(m, 0.0, math.inf)
        x, its, conv, brk = f.solve(rhs), 0, True, False
        cond = None
    else:
        f = factorize_raw(m, d, float(p))
        run = gmres if method == "gmres" else bicgstab
        args = (restart_m,) if method == "gmres" else ()
        x, its, conv, brk = run(m, rhs, f, tol, max_iter, *args)
        cond = condest(f)
    if fwd is not None:
        x = x[fwd]
    rho, res = postprocess(x, D, L)
    return dict(rho=rho, residual=res, iterations=its, converged=conv, breakdown=brk,
                fill=f.fill_factor, condest=cond, perm=fwd, w=w)


def trace_distance(a, b):
    """0.5 * ||a - b||_1 (nuclear norm) for Hermitian a - b."""
    return 0.5 * float(np.sum(np.abs(np.linalg.eigvalsh(a - b))))
