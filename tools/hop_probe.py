"""Dependency-hop latency of the level-ordered sweeps: a bidiagonal system is
one chain (every row waits on the previous one), so sweep time / n is the
publish -> dependent-publish latency.  python tools/hop_probe.py [n] [band]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1504_06768_b200 import factor  # noqa: E402
from paper_1504_06768_b200.sparse import CSRMatrix, from_host  # noqa: E402
from tools.time_grid import ev_time  # noqa: E402


def main(n="20000", band="1"):
    n, band = int(n), int(band)
    rows, cols, vals = [], [], []
    for i in range(n):
        for j in range(max(0, i - band), i + 1):
            rows.append(i)
            cols.append(j)
            vals.append(4.0 + 0j if i == j else -0.5 + 0.1j)
    rp = np.zeros(n + 1, dtype=np.int64)
    np.add.at(rp, np.asarray(rows) + 1, 1)
    rp = np.cumsum(rp)
    A = from_host(CSRMatrix(n, n, rp, np.asarray(cols, dtype=np.int64),
                            np.asarray(vals, dtype=np.complex128)))
    f = factor.factor_batch(A, 0.0, float("inf"))
    f.ensure_levels()
    b = torch.randn(n, dtype=torch.complex128, device="cuda")
    for apw in (1, 2, 4, 16):
        f.Llev.apw = f.Ulev.apw = apw
        ms = ev_time(lambda: factor.solve_lu_levels(f, b), reps=3)
        print(f"n={n} band={band} L levels {f.Llev.nlevels} (G={f.Llev.G}) U levels {f.Ulev.nlevels} "
              f"apw={apw}: apply {ms:.3f} ms -> {ms * 1e6 / f.Llev.nlevels:.0f} ns per L hop")




def timeline(n="20000"):
    """Per-slice stamps of the chain: when the previous slice published, when
    this one saw its sources, when it published."""
    import ctypes
    from paper_1504_06768_b200 import _lib
    n = int(n)
    rp = np.arange(0, 2 * n + 1, 2, dtype=np.int64)
    rp = np.concatenate(([0], np.arange(1, 2 * n, 2)[: n]))
    rows, cols, vals = [0], [0], [4.0 + 0j]
    for i in range(1, n):
        rows += [i, i]
        cols += [i - 1, i]
        vals += [-0.5 + 0.1j, 4.0 + 0j]
    A = from_host(CSRMatrix.from_coo(n, n, rows, cols, vals))
    f = factor.factor_batch(A, 0.0, float("inf"))
    f.ensure_levels()
    f.Llev.apw = f.Ulev.apw = 1
    b = torch.randn(n, dtype=torch.complex128, device="cuda")
    factor.solve_lu_levels(f, b)
    ns = f.Llev.nslices
    buf = torch.zeros(3 * ns, dtype=torch.int64, device="cuda")
    lib = _lib.load()
    lib.rs_debug_slice_times(ctypes.c_void_p(buf.data_ptr()))
    factor.solve_lu_levels(f, b)
    torch.cuda.synchronize()
    lib.rs_debug_slice_times(None)
    t = buf.cpu().numpy().reshape(ns, 3).astype(np.float64)
    t -= t[:, 0].min()
    seen = t[1:, 1] - t[:-1, 2]
    pub = t[1:, 2] - t[1:, 1]
    print(f"chain of {ns} slices: previous published -> sources seen median {np.median(seen):.0f} ns "
          f"(p90 {np.percentile(seen, 90):.0f}); seen -> published median {np.median(pub):.0f} ns "
          f"(p90 {np.percentile(pub, 90):.0f}); start -> seen median {np.median(t[:, 1] - t[:, 0]) / 1e3:.1f} us")
    lib.rs_debug_slice_clock_mode(1)
    buf.zero_()
    lib.rs_debug_slice_times(ctypes.c_void_p(buf.data_ptr()))
    factor.solve_lu_levels(f, b)
    torch.cuda.synchronize()
    lib.rs_debug_slice_times(None)
    lib.rs_debug_slice_clock_mode(0)
    c = buf.cpu().numpy().reshape(ns, 3).astype(np.float64)
    print(f"clock64: key seen -> sources loaded median {np.median(c[1:, 1]):.0f} cycles; "
          f"loaded -> folded median {np.median(c[1:, 0]):.0f}; loaded -> published median "
          f"{np.median(c[1:, 2]):.0f} cycles")
    for s in (1000, 1001, 1002, 1003):
        print(f"  slice {s}: start {t[s, 0]:.0f} seen {t[s, 1]:.0f} end {t[s, 2]:.0f} (prev end {t[s - 1, 2]:.0f})")


if len(sys.argv) > 1 and sys.argv[1] == "timeline":
    timeline(*sys.argv[2:])
    sys.exit(0)

if __name__ == "__main__":
    main(*sys.argv[1:])
