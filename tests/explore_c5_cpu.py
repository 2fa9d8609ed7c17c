"""CPU exploration of the config-5 block-Jacobi preconditioner (not a test;
tests-side because it drives the oracle).  Builds the Kerr x Kerr Liouvillian
at a reduced cutoff, orders it with RCM, factors the diagonal blocks with the
oracle's ILUTP and runs the inverse-power / BiCGStab loop, reporting inner
iteration counts, the triangular-solve DAG depth and factor sizes.

    python tests/explore_c5_cpu.py N blocks d p [max_iter] [floor]
"""
import os
import sys
import time

import numpy as np
import scipy.sparse as sp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402
from paper_1504_06768_b200 import configs  # noqa: E402


def levels_csc(n, cp, ci, lower):
    """DAG depth of a column-oriented triangular solve: level[c] = 1 + max level
    of the columns that update row c."""
    lev = np.zeros(n, dtype=np.int64)
    if lower:
        for c in range(n):
            rows = ci[cp[c] + 1:cp[c + 1]]
            if len(rows):
                np.maximum.at(lev, rows, lev[c] + 1)
    else:
        for c in range(n - 1, -1, -1):
            rows = ci[cp[c]:cp[c + 1] - 1]
            if len(rows):
                np.maximum.at(lev, rows, lev[c] + 1)
    return int(lev.max()) + 1


def main(N=12, blocks=8, d=1e-3, p=2.0, max_iter=1000, floor=0, early=0):
    N, blocks, max_iter, floor = int(N), int(blocks), int(max_iter), float(floor)
    d, p = float(d), float(p)
    t = time.perf_counter()
    H, c = configs.kerr_kerr(N=N)
    L = O.build_liouvillian(H.matrix, [x.matrix for x in c])
    D = N * N
    S = O.shift(L)
    fwd, inv = O.rcm(S)
    A = O.permute(S, fwd)
    P = O.permute(L, fwd)
    n = A.n
    print(f"N={N} n={n} nnz={A.nnz} build {time.perf_counter() - t:.1f}s", flush=True)
    As = sp.csr_matrix((A.v, A.ci, A.rp), shape=(n, n))
    Ps = sp.csr_matrix((P.v, P.ci, P.rp), shape=(n, n))
    bs = -(-n // blocks)
    facs = []
    t = time.perf_counter()
    tot = 0
    for b in range(blocks):
        r0, r1 = b * bs, min(n, (b + 1) * bs)
        Bk = As[r0:r1, r0:r1].tocsr()
        Bk.sort_indices()
        Bc = O.CSR(r1 - r0, r1 - r0, Bk.indptr.astype(np.int64), Bk.indices.astype(np.int64),
                   Bk.data.astype(np.complex128))
        try:
            f = O.factorize_raw(Bc, d, p, pivot_floor=float(floor), early_drop=int(early))
            if f.nfloor:
                print(f"  block {b}: {f.nfloor} substituted pivots", flush=True)
        except O.Breakdown as e:
            print(f"block {b}: {e}")
            return
        facs.append((r0, r1, f))
        tot += len(f.Li) + len(f.Ui)
        if b in (0, blocks // 2):
            print(f"  block {b}: rows {r1 - r0} fill {f.fill_factor:.2f} levels L "
                  f"{levels_csc(f.n, f.Lp, f.Li, True)} U {levels_csc(f.n, f.Up, f.Ui, False)}",
                  flush=True)
    print(f"factor {time.perf_counter() - t:.1f}s nnz(L+U)={tot} ({tot / A.nnz:.2f}x)",
          flush=True)

    def psolve(v):
        out = np.empty_like(v)
        for r0, r1, f in facs:
            out[r0:r1] = f.solve(v[r0:r1])
        return out

    class M:
        solve = staticmethod(psolve)

    class Aop:
        pass

    x = O.start_vector(n, 3)
    x /= np.linalg.norm(x)
    tol = 1e-10
    # oracle bicgstab takes an O.CSR; use it directly (C SpMV)
    for outer in range(1, 8):
        t = time.perf_counter()
        y, its, conv, brk = O.bicgstab(A, x, M, tol / 10, max_iter)
        ny = np.linalg.norm(y)
        y = y / ny
        ov = np.vdot(y, x)
        al = y * (ov / abs(ov))
        diff = np.linalg.norm(al - x)
        rinf = np.max(np.abs(Ps @ y))
        print(f"outer {outer}: inner {its} conv {conv} brk {brk} |y| {ny:.3e} diff {diff:.3e} "
              f"resid_inf {rinf:.3e} ({time.perf_counter() - t:.1f}s)", flush=True)
        x = y
        if diff <= tol or rinf <= tol:
            break


if __name__ == "__main__":
    main(*sys.argv[1:])
