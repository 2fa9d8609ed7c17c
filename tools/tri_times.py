"""Per-row start/publish clocks of the warp-per-row triangular sweeps (c2)."""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1504_06768_b200 import _lib, configs, factor, liouville, ordering  # noqa: E402


def main(cfg="c2", threads="512"):
    c = configs.CONFIGS[cfg]
    H, cops = c["build"]()
    L = liouville.build_liouvillian(H, cops)
    sh = liouville.shift(L)
    fwd, inv = ordering.rcm_device(sh.matrix)
    A = ordering.permute(sh.matrix, fwd, inv)
    f = factor.factor_batch(A, c["d"], c["p"])
    lib = _lib.load()
    fn = lib.rs_debug_tri_probe
    fn.argtypes = [ctypes.c_int] + [ctypes.c_void_p] * 6 + [ctypes.c_int] * 4 + [ctypes.c_void_p]
    lib.rs_debug_tri_times.argtypes = [ctypes.c_void_p]
    n = A.n
    x = torch.randn(n, dtype=torch.complex128, device="cuda")
    out = torch.empty_like(x)
    tt = torch.zeros(2 * n, dtype=torch.int64, device="cuda")
    for which, (rp, ci, v) in ((0, (f.L_rp, f.L_ci, f.L_v)), (1, (f.U_rp, f.U_ci, f.U_v))):
        for rep in range(2):
            lib.rs_debug_tri_times(ctypes.c_void_p(tt.data_ptr()) if rep else None)
            fn(n, rp.data_ptr(), ci.data_ptr(), v.data_ptr(), f.rdiag.data_ptr(), x.data_ptr(),
               out.data_ptr(), which, 1, 1, int(threads), None)
            torch.cuda.synchronize()
        lib.rs_debug_tri_times(None)
        t = tt.view(n, 2).cpu().numpy()
        order = np.arange(n) if which == 0 else np.arange(n)[::-1]
        st, pub = t[order, 0], t[order, 1]
        span = pub.max() - st.min()
        dur = pub - st
        rpn = rp.cpu().numpy()
        cin = ci.cpu().numpy()
        dep = np.array([t[cin[rpn[r]:rpn[r + 1]], 1].max() if rpn[r + 1] > rpn[r] else 0
                        for r in order])
        has = np.array([rpn[r + 1] > rpn[r] for r in order])
        after_dep = (pub - dep)[has]
        late_start = (st - dep)[has]
        print(f"threads={threads} {'LU'[which]}: span {span} cycles = {span / n:.0f}/row; "
              f"row duration median {np.median(dur):.0f}; publish-after-last-source median "
              f"{np.median(after_dep):.0f} p90 {np.percentile(after_dep, 90):.0f}; rows starting "
              f"after their last source {(late_start > 0).mean():.2f}; entries/row "
              f"{np.diff(rpn).mean():.1f}", flush=True)


if __name__ == "__main__":
    main(*sys.argv[1:])
