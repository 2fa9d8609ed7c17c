"""Steady-state drivers: the drop-in surface of the reference steady module
(pkg/src/rhosolve/steady.py:116-260).

Same signatures, defaults, result fields and exceptions as the reference:
`solve_direct`, `solve_iterative`, `inverse_power`, `SteadyStateResult`,
`InnerSolverError`, `PowerIterationError`, `DEFAULT_SEED`, `MAX_OUTER`.
Every stage runs on the GPU through the C ABI: shift / trace modification,
RCM, permutation, LU / ILUTP, then ONE solver launch that runs the whole
inverse-power (or Krylov) iteration on the device, then the unpermute and
post-processing kernels.  Only the seeded start vector (numpy PCG64, as the
reference draws it) and the final rho cross the PCIe bus.

`inverse_power_batch` / `solve_batch` run many independent systems (the
config-4 parameter sweep) as one block-diagonal batch: one CTA per system.
"""

from __future__ import annotations

import os
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib, factor, liouville, ordering
from .liouville import DEFAULT_SIGMA
from .sparse import DeviceCSR

__all__ = ["SteadyStateResult", "solve_direct", "solve_iterative", "inverse_power",
           "inverse_power_batch", "solve_batch", "InnerSolverError", "PowerIterationError",
           "DEFAULT_SEED", "MAX_OUTER", "start_vector"]

DEFAULT_SEED = 12345
MAX_OUTER = 50


class InnerSolverError(RuntimeError):
    """The inner linear solve of the inverse-power iteration produced no
    usable iterate (breakdown or non-finite values)."""


class PowerIterationError(RuntimeError):
    """Inverse-power iteration exceeded the outer iteration budget."""


@dataclass
class SteadyStateResult:
    """Steady-state density matrix plus diagnostics (steady.py:39-59).
    residual = ||L vec(rho)||_2 against the plain Liouvillian."""

    rho: np.ndarray
    method: str
    ordering: str
    residual: float
    iterations: int
    fill_factor: float
    condest: float | None
    build_time: float
    factor_time: float
    solve_time: float
    converged: bool = True
    breakdown: bool = False
    seed: int | None = None
    inner_iterations: int | None = None
    error: str | None = None
    extra: dict = field(default_factory=dict)


_STATS_DT = np.dtype([("status", np.int32), ("outer", np.int32), ("inner_last", np.int32),
                      ("inner_total", np.int32), ("converged", np.int32),
                      ("breakdown", np.int32), ("final_residual", np.float64),
                      ("condest", np.float64)])
assert _STATS_DT.itemsize == _lib.STATS_BYTES


def _sync():
    """Stage boundary for the *_time fields: the current stream only, so work
    queued on the side stream (start-vector upload, plain-matrix permute)
    keeps overlapping the next stage."""
    torch.cuda.current_stream().synchronize()
    return time.perf_counter()


def start_vector(n, seed):
    """steady.py:171-174 (host PCG64 draw, normalised on the device later)."""
    rng = np.random.default_rng(seed)
    return rng.standard_normal(n) + 1j * rng.standard_normal(n)


_POOL = ThreadPoolExecutor(max_workers=1, thread_name_prefix="rhosolve-rng")


_DRAW_THREADS = max(1, int(os.environ.get("RHOSOLVE_DRAW_THREADS", "2")))
_DRAW_POOL = ThreadPoolExecutor(max_workers=_DRAW_THREADS, thread_name_prefix="rhosolve-draw")


def _start_vectors(n, seeds, pin=True):
    """The batch's start vectors drawn straight into pinned host memory, so
    the upload is one asynchronous DMA.  Same bits as start_vector: one
    standard_normal(2n) call continues the PCG64 stream exactly as the
    reference's two calls of n (real part first), and default_rng(seed) is
    Generator(PCG64(seed)); large batches are split over RHOSOLVE_DRAW_THREADS
    threads (default 2: measured on the c4 step, 4 or 8 threads slow the launching thread down more than they shorten the draw)."""
    seeds = list(seeds)
    out = torch.empty(len(seeds) * n, dtype=torch.complex128, pin_memory=pin)
    view = out.numpy().reshape(len(seeds), n)

    def part(lo, hi):
        tmp = np.empty(2 * n)
        for i in range(lo, hi):
            np.random.Generator(np.random.PCG64(seeds[i])).standard_normal(2 * n, out=tmp)
            view[i].real = tmp[:n]
            view[i].imag = tmp[n:]

    m = len(seeds)
    if m >= 64 and _DRAW_THREADS > 1:
        cuts = [m * t // _DRAW_THREADS for t in range(_DRAW_THREADS + 1)]
        futs = [_DRAW_POOL.submit(part, cuts[t], cuts[t + 1]) for t in range(1, _DRAW_THREADS)]
        part(0, cuts[1])
        for fut in futs:
            fut.result()
    else:
        part(0, m)
    return out


_SIDE = {}


def _side_stream(device):
    """A second stream per device for copies and kernels that only the
    solve needs, so they overlap the factorization."""
    st = _SIDE.get(device)
    if st is None:
        st = _SIDE[device] = torch.cuda.Stream(device=device)
    return st


def _upload_start_vectors(n, seeds, device, stream):
    """Draw the start vectors (host thread) and upload them on `stream` as
    soon as they exist, overlapping the factorization; the caller makes its
    stream wait for `stream` before the solve."""
    host = _start_vectors(n, seeds)
    with torch.cuda.stream(stream):
        dev = host.to(device, non_blocking=True)
    return dev, host


def _require_plain(L, values_stream=None):
    if L.variant != "plain":
        raise ValueError(f"expected the plain variant, got {L.variant!r}")
    return liouville.on_device(L, values_stream=values_stream)


def _prepare(system, ordering_name, plain=None, side=None, rcm=None):
    """steady._prepare (steady.py:74-108) on the device.  Returns (matrix,
    rhs, plain_ordered, forward, label, col_fwd): the solution is x[forward]
    (None: unchanged); col_fwd is the column pre-ordering of the factorization
    ('cmd'; None otherwise), see _factor.  `side`: a stream on
    which the plain matrix (read only by the solve) is permuted, overlapping
    the factorization; the caller makes its stream wait for `side` before
    the solve.  rcm: (forward, inverse) already computed for this pattern
    (RCM ignores the diagonal, so the plain matrix's ordering is the shifted
    one's)."""
    m = system.matrix
    if ordering_name == "natural":
        return m, system.rhs, plain, None, "natural", None
    if ordering_name == "rcm":
        fwd, inv = rcm if rcm is not None else ordering.rcm_device(m)
        pm = ordering.permute(m, fwd, inv)
        prhs = None
        if system.rhs is not None:
            prhs = ordering.permute_vector(system.rhs, fwd, m.nsys, m.n, gather=False)
        pp = None
        if plain is not None:
            if side is None:
                pp = ordering.permute(plain, fwd, inv)
            else:
                main = torch.cuda.current_stream(m.values.device)
                side.wait_stream(main)
                with torch.cuda.stream(side):
                    pp = ordering.permute(plain, fwd, inv)
                    for t in (pp.row_ptr, pp.col_idx, pp.values):
                        t.record_stream(main)
                    for t in (fwd, inv, plain.row_ptr, plain.col_idx, plain.values):
                        t.record_stream(side)
        return pm, prhs, pp, fwd, "rcm", None
    if ordering_name == "cmd":
        # MBM rows (when the diagonal is not fully stored) and the minimum-
        # degree column order, both host-native (csrc/cmd_order.cu).  As in
        # the reference (steady.py:95-107) the working matrix, the iterate and
        # the plain matrix stay in the original column coordinates; the
        # column order only feeds the factorization (`colp`, applied by
        # _factor below) and every preconditioner apply ends with x[q] = y.
        (rf, ri, cf, ci), label = ordering.cmd_plan(m)
        pm = ordering.permute_rows_cols(m, ri, None) if ri is not None else m
        prhs = system.rhs
        if system.rhs is not None and rf is not None:
            prhs = ordering.permute_vector(system.rhs, rf, m.nsys, m.n, gather=False)
        return pm, prhs, plain, None, label, cf
    raise ValueError(f"unknown ordering {ordering_name!r}")


def _factor(mat, d, p, col_fwd=None, raise_on_fail=True):
    """factor.lu / factor.ilutp with the optional column pre-ordering of the
    'cmd' path (factor.py:76-78): the column-permuted matrix is factored in
    natural order (bit-identical factors) and the factors remember the
    permutation, which every apply undoes (x[q] = y, factor.py:147-148)."""
    if col_fwd is None:
        return factor.factor_batch(mat, d, p, raise_on_fail=raise_on_fail)
    f = factor.factor_batch(ordering.permute_rows_cols(mat, None, col_fwd), d, p,
                            raise_on_fail=raise_on_fail)
    f.colp_dev = col_fwd
    from .sparse import Permutation
    f.colp = Permutation(col_fwd[:mat.n].cpu().numpy().astype(np.int64))
    return f


_grid_min_n = factor.grid_min_n


def _solve_grid(mode, A, P, f, rhs, tol, max_iter, restart_m, want_condest):
    """One cooperative launch over the whole GPU.  f may be a batch of
    block-Jacobi factors (f.nsys blocks of order f.n tiling the n rows of A)."""
    import ctypes
    dev = A.values.device
    n = A.n
    x = torch.empty(n, dtype=torch.complex128, device=dev)
    stats = torch.zeros(_STATS_DT.itemsize, dtype=torch.uint8, device=dev)
    a = _lib.GridArgs()
    a.n, a.nb, a.mode = n, n, mode
    a.A_rp, a.A_ci, a.A_v = A.row_ptr.data_ptr(), A.col_idx.data_ptr(), A.values.data_ptr()
    if P is not None:
        a.P_rp, a.P_ci, a.P_v = P.row_ptr.data_ptr(), P.col_idx.data_ptr(), P.values.data_ptr()
    if f is not None:
        if f.nsys * f.n != n:
            raise ValueError("preconditioner blocks do not tile the system")
        f.ensure_levels()
        a.nb = f.n
        f.Llev.fill(a.L)
        f.Ulev.fill(a.U)
        a.rdiag, a.pinv = f.rdiag.data_ptr(), f.pinv.data_ptr()
        if f.colp_dev is not None:
            a.colp = f.colp_dev.data_ptr()
    a.rhs, a.x, a.stats = rhs.data_ptr(), x.data_ptr(), stats.data_ptr()
    a.tol, a.max_iter, a.restart_m = float(tol), int(max_iter), int(restart_m)
    a.max_outer, a.want_condest = MAX_OUTER, 1 if want_condest else 0
    _lib.call("rs_grid_solve", ctypes.byref(a), _lib.stream_ptr())
    st = np.frombuffer(stats.cpu().numpy().tobytes(), dtype=_STATS_DT)
    return x, st


def _wide(f):
    """True when the factors' dependency DAG is wide enough for the grid-wide
    level sweeps.  A hop between SMs costs ~2 us (tools/hop_probe.py), the
    one-warp column sweep of colsweep.cuh ~1.4 us per column, so a chain-like
    DAG (config 3: ~350 entries per row, ~3 rows per level) is faster on one
    CTA; sparse factors (config 5: ~9 entries per row, thousands of rows per
    level) belong on the grid.  Decided from the mean row length, which needs
    no analysis pass; RHOSOLVE_GRID_FORCE=1/0 overrides."""
    import os
    force = os.environ.get("RHOSOLVE_GRID_FORCE")
    if force is not None:
        return force != "0"
    if f is None:
        return True
    return float(np.sum(f.lnnz + f.unnz)) / (f.nsys * f.n) < 64.0


def _solve(mode, A, P, f, rhs, tol, max_iter, restart_m, want_condest, threads=0, trace=None):
    dev = A.values.device
    B, n = A.nsys, A.n
    if B == 1 and n >= _grid_min_n() and trace is None and (f is None or f.ok) and _wide(f):
        return _solve_grid(mode, A, P, f, rhs, tol, max_iter, restart_m, want_condest)
    if not threads:
        # one CTA per system: big batches use 4-warp CTAs so four systems stay
        # resident per SM (one wave for the 512-instance sweep); a lone system
        # gets 8 warps and the 255-register kernel (the column-sweep consumer
        # then runs without spills)
        threads = 128 if B > 148 else 256
    x = torch.empty(B * n, dtype=torch.complex128, device=dev)
    stats = torch.zeros(B * _STATS_DT.itemsize, dtype=torch.uint8, device=dev)
    a = _lib.SolverArgs()
    a.n, a.nsys, a.mode, a.threads = n, B, mode, threads
    a.A_rp, a.A_ci, a.A_v = A.row_ptr.data_ptr(), A.col_idx.data_ptr(), A.values.data_ptr()
    if P is not None:
        a.P_rp, a.P_ci, a.P_v = P.row_ptr.data_ptr(), P.col_idx.data_ptr(), P.values.data_ptr()
    if f is not None:
        if f.csc:  # column streams, reference column sweeps on shared memory
            f.ensure_cols()
            (lo, li, lv, lm, _), (uo, ui, uv, um, ur) = f.Ls, f.Us
            a.Ls_rowoff, a.Ls_idx, a.Ls_val, a.Ls_meta = (_lib.ptr(lo), _lib.ptr(li),
                                                          _lib.ptr(lv), _lib.ptr(lm))
            a.Us_rowoff, a.Us_idx, a.Us_val, a.Us_meta, a.Us_rd = (
                _lib.ptr(uo), _lib.ptr(ui), _lib.ptr(uv), _lib.ptr(um), _lib.ptr(ur))
            a.col_reach = int(f.reach)
        else:
            f.ensure_rows()
            a.L_rp, a.L_ci, a.L_v = f.L_rp.data_ptr(), f.L_ci.data_ptr(), f.L_v.data_ptr()
            a.U_rp, a.U_ci, a.U_v = f.U_rp.data_ptr(), f.U_ci.data_ptr(), f.U_v.data_ptr()
        a.rdiag, a.pinv = f.rdiag.data_ptr(), f.pinv.data_ptr()
        if f.colp_dev is not None:  # every apply ends with x[q] = y (factor.py:147-148)
            a.colp = f.colp_dev.data_ptr()
        if not f.ok:  # systems whose factorization failed are masked out
            a.skip = f.fail_dev.data_ptr()
    a.rhs, a.x, a.stats = rhs.data_ptr(), x.data_ptr(), stats.data_ptr()
    a.tol, a.max_iter, a.restart_m = float(tol), int(max_iter), int(restart_m)
    a.max_outer, a.want_condest = MAX_OUTER, 1 if want_condest else 0
    if trace is not None:  # residual history of system 0 (krylov.py:62-64)
        tbuf = torch.zeros(2 * (int(max_iter) + 2), dtype=torch.float64, device=dev)
        tcnt = torch.zeros(1, dtype=torch.int32, device=dev)
        a.trace, a.trace_count, a.trace_cap = tbuf.data_ptr(), tcnt.data_ptr(), int(max_iter) + 2
    import ctypes
    _lib.call("rs_steady_solve", ctypes.byref(a), _lib.stream_ptr())
    st = np.frombuffer(stats.cpu().numpy().tobytes(), dtype=_STATS_DT)
    if trace is not None:
        rows = tbuf.cpu().numpy().reshape(-1, 2)[:min(int(tcnt.item()), int(max_iter) + 2)]
        for it, res in rows:
            trace.write(f"{int(it)},{res:.17g}\n")
    return x, st


def _postprocess(x, fwd, L):
    M = L.matrix
    D = L.hilbert_dim
    dev = M.values.device
    rho = torch.empty(M.nsys * D * D, dtype=torch.complex128, device=dev)
    res = torch.empty(M.nsys, dtype=torch.float64, device=dev)
    _lib.call("rs_postprocess", M.nsys, D, _lib.ptr(x), _lib.ptr(fwd), _lib.ptr(M.row_ptr),
              _lib.ptr(M.col_idx), _lib.ptr(M.values), _lib.ptr(rho), _lib.ptr(res), None,
              _lib.stream_ptr())
    # one D2H into pinned host memory (torch caches pinned blocks)
    out = torch.empty(rho.numel() + M.nsys * 2, dtype=torch.complex128, pin_memory=True)
    out[:rho.numel()].copy_(rho, non_blocking=True)
    out[rho.numel():].view(torch.float64)[:M.nsys].copy_(res, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    on = out.numpy()
    return (on[:rho.numel()].reshape(M.nsys, D, D).copy(),
            on[rho.numel():].view(np.float64)[:M.nsys].copy())


def _check_ops(tol=None, max_iter=None, restart_m=None):
    if tol is not None and not tol > 0:
        raise ValueError("tol must be > 0")
    if max_iter is not None and max_iter < 1:
        raise ValueError("max_iter must be >= 1")
    if restart_m is not None and restart_m < 1:
        raise ValueError("restart_m must be >= 1")


# ------------------------------------------------------------------ API ----
def solve_direct(L, ordering_name="natural", w=None):
    """Steady state by one complete-LU solve of the trace-modified system
    (steady.py:116-134)."""
    L = _require_plain(L)
    t0 = _sync()
    modified = liouville.build_modified(L, w)
    mat, rhs, _, fwd, label, colf = _prepare(modified, ordering_name)
    t1 = _sync()
    f = _factor(mat, 0.0, float("inf"), colf)
    t2 = _sync()
    x, _ = _solve(_lib.LIN_DIRECT, mat, None, f, rhs, 1.0, 1, 1, False)
    rho, res = _postprocess(x, fwd, L)
    t3 = _sync()
    return SteadyStateResult(rho=rho[0], method="direct", ordering=label, residual=float(res[0]),
                             iterations=0, fill_factor=f.fill_factor, condest=None,
                             build_time=t1 - t0, factor_time=t2 - t1, solve_time=t3 - t2)


def solve_iterative(L, ordering_name="natural", solver="gmres", d=1e-4, p=300.0, tol=1e-14,
                    restart_m=20, max_iter=1000, w=None):
    """Preconditioned Krylov on the trace-modified system (steady.py:137-168).
    Non-convergence and solver breakdown are reported, not raised."""
    L = _require_plain(L)
    if solver not in ("gmres", "bicgstab"):
        raise ValueError(f"unknown solver {solver!r}")
    _check_ops(tol, max_iter, restart_m)
    t0 = _sync()
    modified = liouville.build_modified(L, w)
    if d < 0:
        raise ValueError("drop tolerance d must be >= 0")
    if not p >= 1:
        raise ValueError("fill limit p must be >= 1")
    mat, rhs, _, fwd, label, colf = _prepare(modified, ordering_name)
    t1 = _sync()
    f = _factor(mat, float(d), float(p), colf)
    t2 = _sync()
    mode = _lib.LIN_GMRES if solver == "gmres" else _lib.LIN_BICGSTAB
    x, st = _solve(mode, mat, None, f, rhs, tol, max_iter, restart_m, True)
    rho, res = _postprocess(x, fwd, L)
    t3 = _sync()
    s = st[0]
    return SteadyStateResult(rho=rho[0], method=f"iterative-{solver}", ordering=label,
                             residual=float(res[0]), iterations=int(s["inner_last"]),
                             fill_factor=f.fill_factor, condest=float(s["condest"]),
                             build_time=t1 - t0, factor_time=t2 - t1, solve_time=t3 - t2,
                             converged=bool(s["converged"]), breakdown=bool(s["breakdown"]),
                             extra={"final_residual": float(s["final_residual"])})


_STATUS_MSG = {
    _lib.SOLVE_INNER_BREAKDOWN: (InnerSolverError, "inner Krylov solve broke down; try a "
                                 "smaller drop tolerance or a larger fill budget"),
    _lib.SOLVE_INNER_NONFINITE: (InnerSolverError, "inner Krylov solve broke down; try a "
                                 "smaller drop tolerance or a larger fill budget"),
    _lib.SOLVE_INNER_NO_PROGRESS: (InnerSolverError, "inner Krylov solve made no progress"),
    _lib.SOLVE_UNUSABLE_VECTOR: (InnerSolverError, "inner solve returned an unusable vector"),
    _lib.SOLVE_POWER_NOT_CONVERGED: (PowerIterationError,
                                     f"no convergence within {MAX_OUTER} outer iterations"),
}


def _power_core(L, sigma, tol, inner, ordering_name, solver, d, p, restart_m, max_iter, seeds,
                raise_errors, threads=0):
    m = L.matrix
    device = (m.values.device if isinstance(m, DeviceCSR)
              else torch.device("cuda", torch.cuda.current_device()))
    side = _side_stream(device)
    # host batches upload their values on the side stream: the RCM below
    # needs only the pattern and overlaps that copy
    L = _require_plain(L, values_stream=side)
    if inner not in ("direct", "iterative"):
        raise ValueError(f"unknown inner solve {inner!r}")
    if not tol > 0:
        raise ValueError("tol must be > 0")
    # like the reference (steady.py:210), any solver name other than "gmres"
    # selects BiCGStab
    _check_ops(None, max_iter, restart_m)
    t0 = _sync()
    # the seeded start vectors (numpy PCG64, drawn exactly as steady.py:171-174)
    # are generated on a host thread while the GPU orders and factors
    x0_future = _POOL.submit(_upload_start_vectors, L.n, list(seeds), device, side)
    # RCM of the plain pattern = RCM of the shifted one (the graph drops
    # self-loops, and shifting only adds diagonal entries: ordering.py:62-79)
    rcm = ordering.rcm_device(L.matrix) if ordering_name == "rcm" else None
    torch.cuda.current_stream(device).wait_stream(side)  # the values have landed
    shifted = liouville.shift(L, sigma)
    mat, _, plain, fwd, label, colf = _prepare(shifted, ordering_name, plain=L.matrix,
                                               side=side, rcm=rcm)
    if plain is None:
        plain = L.matrix
    t1 = _sync()
    if inner == "direct":
        f = _factor(mat, 0.0, float("inf"), colf, raise_on_fail=raise_errors)
        mode = _lib.INV_DIRECT
    else:
        if d < 0:
            raise ValueError("drop tolerance d must be >= 0")
        if not p >= 1:
            raise ValueError("fill limit p must be >= 1")
        f = _factor(mat, float(d), float(p), colf, raise_on_fail=raise_errors)
        mode = _lib.INV_GMRES if solver == "gmres" else _lib.INV_BICGSTAB
    t2 = _sync()
    x0, _host = x0_future.result()
    main = torch.cuda.current_stream(device)
    main.wait_stream(side)  # the start vectors and the permuted plain matrix
    x0.record_stream(main)
    if not f.ok and not f.solvable:  # nothing of the batch can be solved
        return None, f, None, None, label, (t0, t1, t2, _sync())
    x, st = _solve(mode, mat, plain, f, x0, tol, max_iter, restart_m, inner == "iterative",
                   threads)
    rho, res = _postprocess(x, fwd, L)
    t3 = _sync()
    return (rho, res), f, st, x, label, (t0, t1, t2, t3)


def inverse_power(L, sigma=DEFAULT_SIGMA, tol=1e-14, inner="direct", ordering_name="natural",
                  solver="gmres", d=1e-4, p=300.0, restart_m=20, max_iter=1000,
                  seed=DEFAULT_SEED):
    """Null eigenvector of the shifted Liouvillian by inverse-power iteration
    (steady.py:177-260); inner="iterative" is the paper's doubly-iterative
    method (ILUTP-preconditioned BiCGStab/GMRES to tol/10 each outer step)."""
    if L.nsys != 1:
        raise ValueError("inverse_power takes one system; use inverse_power_batch")
    out, f, st, _, label, (t0, t1, t2, t3) = _power_core(
        L, sigma, tol, inner, ordering_name, solver, d, p, restart_m, max_iter, [seed], True)
    s = st[0]
    if s["status"] != _lib.SOLVE_OK:
        exc, msg = _STATUS_MSG[int(s["status"])]
        raise exc(msg)
    rho, res = out
    return SteadyStateResult(
        rho=rho[0], method="power-direct" if inner == "direct" else "power-doubly-iterative",
        ordering=label, residual=float(res[0]), iterations=int(s["outer"]),
        fill_factor=f.fill_factor, condest=float(s["condest"]) if inner == "iterative" else None,
        build_time=t1 - t0, factor_time=t2 - t1, solve_time=t3 - t2, seed=seed,
        inner_iterations=int(s["inner_total"]) if inner == "iterative" else None)


def inverse_power_batch(L, seeds, sigma=DEFAULT_SIGMA, tol=1e-14, inner="direct",
                        ordering_name="natural", solver="gmres", d=1e-4, p=300.0,
                        restart_m=20, max_iter=1000, threads=0):
    """inverse_power over every system of a block-diagonal batch in one pass
    (one CTA per system).  Per-system failures are reported on the result's
    `error` field instead of raising."""
    seeds = list(seeds)
    if len(seeds) != L.nsys:
        raise ValueError("one seed per system required")
    out, f, st, _, label, (t0, t1, t2, t3) = _power_core(
        L, sigma, tol, inner, ordering_name, solver, d, p, restart_m, max_iter, seeds, False,
        threads)
    results = []
    method = "power-direct" if inner == "direct" else "power-doubly-iterative"
    fills = np.asarray(f.fill_factors, dtype=np.float64).tolist()
    fail = f.fail.tolist()
    bt, ft = t1 - t0, t2 - t1

    def failed(b, msg):
        return SteadyStateResult(
            rho=None, method=method, ordering=label, residual=float("nan"), iterations=0,
            fill_factor=fills[b], condest=None, build_time=bt, factor_time=ft, solve_time=0.0,
            converged=False, seed=seeds[b], error=msg)

    if out is None:  # no system could be solved: every entry carries the reason
        for b in range(L.nsys):
            results.append(failed(b, _factor_error(fail[b])))
        return results
    # per-system fields as Python lists once (structured-array element access
    # per system costs more than the solve of a small system)
    rho, resid = out
    resid = resid.tolist()
    status = st["status"].tolist()
    outer = st["outer"].tolist()
    it = inner == "iterative"
    cond = st["condest"].tolist() if it else None
    inner_tot = st["inner_total"].tolist() if it else None
    stime = t3 - t2
    for b in range(L.nsys):
        if status[b] == _lib.SOLVE_SKIPPED:  # only this system is lost
            results.append(failed(b, _factor_error(fail[b])))
            continue
        err = None if status[b] == _lib.SOLVE_OK else _STATUS_MSG[int(status[b])][1]
        results.append(SteadyStateResult(
            rho=rho[b], method=method, ordering=label, residual=resid[b],
            iterations=outer[b], fill_factor=fills[b],
            condest=cond[b] if it else None,
            build_time=bt, factor_time=ft, solve_time=stime, seed=seeds[b],
            inner_iterations=inner_tot[b] if it else None, error=err))
    return results


def _factor_error(step):
    if step >= 0:
        return f"zero pivot at elimination step {int(step)}"
    return "not solved: another system of the batch failed to factor"


def solve_batch(L, method="bicgstab", ordering_name="natural", d=1e-4, p=300.0, tol=1e-14,
                restart_m=20, max_iter=1000, w=None, threads=0):
    """solve_iterative / solve_direct (method="direct") over a batch.  A
    system whose factorization hits a zero pivot is reported on its result's
    `error` field; the others are solved."""
    if method not in ("direct", "gmres", "bicgstab"):
        raise ValueError(f"unknown method {method!r}")
    L = _require_plain(L)
    _check_ops(tol, max_iter, restart_m)
    t0 = _sync()
    modified = liouville.build_modified(L, w)
    mat, rhs, _, fwd, label, colf = _prepare(modified, ordering_name)
    t1 = _sync()
    if method == "direct":
        f = _factor(mat, 0.0, float("inf"), colf, raise_on_fail=False)
        mode = _lib.LIN_DIRECT
    else:
        f = _factor(mat, float(d), float(p), colf, raise_on_fail=False)
        mode = _lib.LIN_GMRES if method == "gmres" else _lib.LIN_BICGSTAB
    t2 = _sync()
    name = "direct" if method == "direct" else f"iterative-{method}"
    fail = f.fail.tolist()

    def failed(b):
        return SteadyStateResult(
            rho=None, method=name, ordering=label, residual=float("nan"), iterations=0,
            fill_factor=float(f.fill_factors[b]), condest=None, build_time=t1 - t0,
            factor_time=t2 - t1, solve_time=0.0, converged=False, error=_factor_error(fail[b]))

    if not f.ok and not f.solvable:
        return [failed(b) for b in range(L.nsys)]
    x, st = _solve(mode, mat, None, f, rhs, tol, max_iter, restart_m, method != "direct",
                   threads)
    rho, res = _postprocess(x, fwd, L)
    t3 = _sync()
    return [failed(b) if st[b]["status"] == _lib.SOLVE_SKIPPED else
            SteadyStateResult(rho=rho[b], method=name, ordering=label, residual=float(res[b]),
                              iterations=int(st[b]["inner_last"]),
                              fill_factor=float(f.fill_factors[b]),
                              condest=None if method == "direct" else float(st[b]["condest"]),
                              build_time=t1 - t0, factor_time=t2 - t1, solve_time=t3 - t2,
                              converged=bool(st[b]["converged"]),
                              breakdown=bool(st[b]["breakdown"]))
            for b in range(L.nsys)]
