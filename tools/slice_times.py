"""Per-slice timeline of the level-ordered L sweep (tuning).
    python tools/slice_times.py c3|c5 [args]"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1504_06768_b200 import _lib, configs, factor, liouville, ordering  # noqa: E402


def main(which="c3", p="300"):
    if which == "c3":
        L = liouville.build_liouvillian(*configs.optomech())
        d, p = 1e-4, float(p)
    else:
        L = liouville.build_liouvillian(*configs.jc_rwa())
        d, p = 1e-4, 300.0
    S = liouville.shift(L)
    fwd, inv = ordering.rcm_device(S.matrix)
    A = ordering.permute(S.matrix, fwd, inv)
    f = factor.factor_batch(A, d, p)
    f.ensure_levels()
    b = torch.randn(A.n, dtype=torch.complex128, device="cuda")
    factor.solve_lu_levels(f, b)
    ns = f.Llev.nslices
    buf = torch.zeros(3 * ns, dtype=torch.int64, device="cuda")
    lib = _lib.load()
    lib.rs_debug_slice_times(ctypes.c_void_p(buf.data_ptr()))
    factor.solve_lu_levels(f, b)
    torch.cuda.synchronize()
    lib.rs_debug_slice_times(None)
    t = buf.cpu().numpy().reshape(ns, 3).astype(np.float64)
    t0 = t[:, 0].min()
    t -= t0
    print(f"slices {ns} G={f.Llev.G} apw={f.Llev.apw} levels {f.Llev.nlevels}; L sweep span "
          f"{t[:, 2].max() / 1e3:.1f} us")
    dur = t[:, 2] - t[:, 0]
    first = t[:, 1] - t[:, 0]
    gap = np.diff(np.sort(t[:, 2]))
    print(f"per-slice duration median {np.median(dur) / 1e3:.2f} us p90 {np.percentile(dur, 90) / 1e3:.2f}; "
          f"first step median {np.median(first) / 1e3:.2f} us; completion gap median "
          f"{np.median(gap):.0f} ns mean {gap.mean():.0f} ns")
    for s in (0, 1, 2, 10, 100, 1000, ns // 2, ns // 2 + 1, ns - 2, ns - 1):
        if s < ns:
            print(f"  slice {s}: start {t[s, 0] / 1e3:.1f} first {t[s, 1] / 1e3:.1f} end {t[s, 2] / 1e3:.1f} us")
    w = (f.Llev.sptr[1:] - f.Llev.sptr[:-1]).cpu().numpy() // 32
    print(f"steps per slice: median {np.median(w)} max {w.max()}")


if __name__ == "__main__":
    main(*sys.argv[1:])
