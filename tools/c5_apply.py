"""c5 block-Jacobi factors: analysis, apply and SpMV timings (tuning).
    python tools/c5_apply.py N blocks d p"""
import ctypes
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1504_06768_b200 import _lib, configs, factor, liouville, ordering, sharded  # noqa: E402
from tools.time_grid import apply_stats, spmv_stats, ev_time  # noqa: E402


def main(N="20", blocks="16", d="1e-2", p="2"):
    N, blocks, d, p = int(N), int(blocks), float(d), float(p)
    L = liouville.build_liouvillian(*configs.kerr_kerr(N=N))
    S = liouville.shift(L)
    fwd, inv = ordering.rcm_device(S.matrix)
    A = ordering.permute(S.matrix, fwd, inv)
    n = A.n
    spmv_stats(A, f"c5 N={N}")
    t = time.perf_counter()
    M = sharded._block_jacobi((A.row_ptr, A.col_idx, A.values), 0, n, n // blocks, d, p, 1.0, True)
    torch.cuda.synchronize()
    print(f"factor {time.perf_counter() - t:.2f}s nfloor {M.nfloor.tolist()}", flush=True)
    t = time.perf_counter()
    M.ensure_rows()
    torch.cuda.synchronize()
    print(f"rows {time.perf_counter() - t:.3f}s", flush=True)
    for up in (False, True):
        t = time.perf_counter()
        tl = factor._tri_levels(M, up)
        torch.cuda.synchronize()
        print(f"levels upper={up}: {time.perf_counter() - t:.3f}s nlev {tl.nlevels} G {tl.G} apw {tl.apw} "
              f"slices {tl.nslices} entries {tl.entries}", flush=True)
        w = (tl.sptr[1:] - tl.sptr[:-1]).cpu().numpy() // 32
        print(f"   steps/slice median {np.median(w)} mean {w.mean():.1f} max {w.max()}", flush=True)
    apply_stats(M, f"c5 N={N} blocks={blocks}")
    b = torch.randn(n, dtype=torch.complex128, device="cuda")
    for mode in ("0", "1", "0", "1"):
        os.environ["RHOSOLVE_TRI_MODE"] = mode
        for apw in (2, 4, 8, 16):
            M.Llev.apw = M.Ulev.apw = apw
            ms = ev_time(lambda: factor.solve_lu_levels(M, b), reps=3)
            print(f"  mode={mode} apw={apw}: apply {ms:.3f} ms", flush=True)
    os.environ["RHOSOLVE_TRI_MODE"] = "0"
    M.Llev.apw = M.Ulev.apw = 4
    # slice timeline of the L sweep
    ns = M.Llev.nslices
    buf = torch.zeros(3 * ns, dtype=torch.int64, device="cuda")
    lib = _lib.load()
    lib.rs_debug_slice_times(ctypes.c_void_p(buf.data_ptr()))
    factor.solve_lu_levels(M, b)
    torch.cuda.synchronize()
    lib.rs_debug_slice_times(None)
    tt = buf.cpu().numpy().reshape(ns, 3).astype(np.float64)
    tt -= tt[:, 0].min()
    dur = tt[:, 2] - tt[:, 0]
    wait = tt[:, 1] - tt[:, 0]
    print(f"L sweep span {tt[:, 2].max() / 1e3:.1f} us; slice duration median {np.median(dur) / 1e3:.2f} "
          f"p90 {np.percentile(dur, 90) / 1e3:.2f} us; wait median {np.median(wait) / 1e3:.2f} us")
    H = 32 // M.Llev.G
    first_row = M.Llev.order[::H].cpu().numpy()
    lev = M.Llev.level.cpu().numpy()[np.maximum(first_row, 0)]
    nl = M.Llev.nlevels
    lev_end = np.zeros(nl)
    np.maximum.at(lev_end, lev, tt[:, 2])
    lev_cnt = np.bincount(lev, minlength=nl)
    dt = np.diff(np.maximum.accumulate(lev_end))
    for a, b in ((0, 50), (50, 150), (150, 300), (300, 400), (400, nl - 1)):
        b = min(b, nl - 1)
        if a < b:
            print(f"   levels {a}-{b}: {lev_cnt[a:b].mean():.0f} slices/level, "
                  f"{dt[a:b].mean() / 1e3:.2f} us per level (max {dt[a:b].max() / 1e3:.1f})")
    ends = np.sort(tt[:, 2])
    for q in (0.1, 0.25, 0.5, 0.75, 0.9, 1.0):
        print(f"   {int(q * 100)}% of slices done at {ends[int(q * (ns - 1))] / 1e3:.1f} us")


if __name__ == "__main__":
    main(*sys.argv[1:])
