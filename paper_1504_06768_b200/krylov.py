"""Preconditioned GMRES(m) and BiCGStab on the GPU: the drop-in for the
reference krylov module (pkg/src/rhosolve/krylov.py:24-291).

Each call is one launch of the device-resident solver (csrc/solver.cu) with
the reference control flow (monitor on the preconditioned residual,
true-residual confirmation, stall exit, breakdown flags).  `trace` (a text
stream, krylov.py:62-64) receives the same "iteration,residual" rows as the
reference's: the kernel records them on the device and they are written out
after the solve.  A preconditioner built with a column pre-ordering
(factor.ilutp(col_perm=...)) is applied with its x[q] = y scatter
(factor.py:147-148), as krylov's solve_lu calls do."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

__all__ = ["IterOptions", "IterResult", "gmres", "bicgstab"]


@dataclass
class IterOptions:
    """tol is the relative L2 residual target (krylov.py:24-39)."""

    tol: float = 1e-10
    max_iter: int = 1000
    restart_m: int = 20
    preconditioner: object = None

    def check(self):
        if not self.tol > 0:
            raise ValueError("tol must be > 0")
        if self.max_iter < 1:
            raise ValueError("max_iter must be >= 1")
        if self.restart_m < 1:
            raise ValueError("restart_m must be >= 1")


@dataclass
class IterResult:
    """krylov.py:42-51; final_residual = ||b - A x||_2 at exit."""

    x: object
    iterations: int
    final_residual: float
    converged: bool
    breakdown: bool


def _run(mode, a, b, opts, trace=None):
    from .steady import _solve  # shared launcher
    A = a.matrix if hasattr(a, "matrix") else a
    opts = opts if opts is not None else IterOptions()
    opts.check()
    host = not isinstance(b, torch.Tensor)
    bt = (torch.from_numpy(np.ascontiguousarray(b, dtype=np.complex128)).to(A.values.device)
          if host else b.to(torch.complex128).contiguous())
    if bt.numel() != A.n * A.nsys:
        raise ValueError("system must be square with matching rhs length")
    x, st = _solve(mode, A, None, opts.preconditioner, bt, opts.tol, opts.max_iter,
                   opts.restart_m, False, trace=trace)
    s = st[0]
    return IterResult(x.cpu().numpy() if host else x, int(s["inner_last"]),
                      float(s["final_residual"]), bool(s["converged"]), bool(s["breakdown"]))


def gmres(a, b, opts=None, trace=None):
    """Restarted GMRES(m), left-preconditioned, x0 = 0 (krylov.py:67-178)."""
    return _run(_lib.LIN_GMRES, a, b, opts, trace)


def bicgstab(a, b, opts=None, trace=None):
    """Left-preconditioned BiCGStab, x0 = 0 (krylov.py:181-291)."""
    return _run(_lib.LIN_BICGSTAB, a, b, opts, trace)
