"""Timing of the grid-wide path.
    python tools/time_grid.py c3 [solver=bicgstab|gmres|direct] [p=300]
    python tools/time_grid.py c5 N blocks d p [max_iter] [floor]
Prints per-stage times, iteration counts, the plain-L residual and the
achieved algorithmic GB/s of the level-ordered apply and of the SpMV."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1504_06768_b200 import _lib, configs, factor, liouville, ordering, sharded, steady  # noqa: E402


def ev_time(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def apply_stats(f, tag):
    N = f.nsys * f.n
    b = torch.randn(N, dtype=torch.complex128, device="cuda")
    t0 = time.perf_counter()
    f.ensure_levels()
    torch.cuda.synchronize()
    t_an = time.perf_counter() - t0
    ms = ev_time(lambda: factor.solve_lu_levels(f, b))
    nnz = float(np.sum(f.lnnz + f.unnz))
    algo = 20.0 * nnz + 72.0 * N
    print(f"{tag}: levels L {f.Llev.nlevels} (G={f.Llev.G}) U {f.Ulev.nlevels} (G={f.Ulev.G}) "
          f"analysis {t_an * 1e3:.1f} ms; apply {ms:.3f} ms = {algo / ms / 1e6:.1f} GB/s "
          f"algorithmic ({algo / 1e6:.1f} MB; stored {20 * (f.Llev.entries + f.Ulev.entries) / 1e6:.1f} MB)",
          flush=True)


def spmv_stats(A, tag):
    x = torch.randn(A.n * A.nsys, dtype=torch.complex128, device="cuda")
    y = torch.empty_like(x)
    ms = ev_time(lambda: _lib.call("rs_csr_matvec", A.nsys, A.n, _lib.ptr(A.row_ptr),
                                   _lib.ptr(A.col_idx), _lib.ptr(A.values), _lib.ptr(x),
                                   _lib.ptr(y), _lib.stream_ptr()))
    algo = 20.0 * A.nnz + 4.0 * (A.n * A.nsys + 1) + 32.0 * A.n * A.nsys
    print(f"{tag}: SpMV {ms:.3f} ms = {algo / ms / 1e6:.1f} GB/s algorithmic ({algo / 1e6:.1f} MB)",
          flush=True)


def c3(solver="bicgstab", p="300"):
    p = float(p)
    H, c = configs.optomech()
    L = liouville.build_liouvillian(H, c)
    for rep in range(2):
        if solver == "direct":
            r = steady.solve_direct(L, "rcm")
        else:
            r = steady.inverse_power(L, tol=1e-12, inner="iterative", ordering_name="rcm",
                                     solver=solver, restart_m=20, d=1e-4, p=p)
        print(f"c3 {solver} p={p}: build {r.build_time:.3f}s factor {r.factor_time:.3f}s solve "
              f"{r.solve_time:.3f}s outer {r.iterations} inner {r.inner_iterations} residual "
              f"{r.residual:.2e} fill {r.fill_factor:.2f}", flush=True)
    S = liouville.shift(L)
    fwd, inv = ordering.rcm_device(S.matrix)
    A = ordering.permute(S.matrix, fwd, inv)
    spmv_stats(A, "c3")
    f = factor.factor_batch(A, 1e-4, p)
    apply_stats(f, f"c3 ILUTP(1e-4,{p})")


def c5(N="20", blocks="8", d="1e-2", p="2", max_iter="1000", floor="0", early="0"):
    N, blocks, max_iter = int(N), int(blocks), int(max_iter)
    d, p, floor = float(d), float(p), float(floor)
    t = time.perf_counter()
    H, c = configs.kerr_kerr(N=N)
    L = liouville.build_liouvillian(H, c)
    torch.cuda.synchronize()
    print(f"c5 N={N} n={L.n} nnz={L.matrix.nnz} assembly(+host ops) {time.perf_counter() - t:.2f}s",
          flush=True)
    r = sharded.inverse_power_sharded(L, tol=1e-10, d=d, p=p, seed=3, blocks=blocks,
                                      max_iter=max_iter, pivot_floor=floor, early_drop=bool(int(early)),
                                      log=lambda m: print(m, flush=True))
    print(f"c5: build {r.build_time:.2f}s factor {r.factor_time:.2f}s solve {r.solve_time:.2f}s "
          f"outer {r.iterations} inner {r.inner_iterations} residual {r.residual:.3e} "
          f"fill {r.fill_factor:.2f} extra {r.extra}", flush=True)
    tr = np.trace(r.rho)
    print(f"c5: trace {tr:.6f} hermitian err {np.abs(r.rho - r.rho.conj().T).max():.2e}",
          flush=True)


if __name__ == "__main__":
    {"c3": c3, "c5": c5}[sys.argv[1]](*sys.argv[2:])
