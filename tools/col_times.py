"""Per-row consumer clocks of the column sweep (L of system 0), tuning."""
import ctypes
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1504_06768_b200 import _lib, configs, factor, liouville, ordering  # noqa: E402


def main(cfg="c4"):
    if cfg == "c4":
        L = liouville.build_liouvillian(*configs.jc_sweep(0))
        d, p = 0.0, math.inf
    else:
        c = configs.CONFIGS[cfg]
        L = liouville.build_liouvillian(*c["build"]())
        d, p = c["d"], c["p"]
    sh = liouville.shift(L)
    fwd, inv = ordering.rcm_device(sh.matrix)
    A = ordering.permute(sh.matrix, fwd, inv)
    f = factor.factor_batch(A, d, p)
    rows = int(f.Ls[0][-1].item())
    buf = torch.zeros(3 * rows + 16, dtype=torch.int64, device="cuda")
    lib = _lib.load()
    lib.rs_debug_col_times.argtypes = [ctypes.c_void_p]
    x = torch.randn(A.n, dtype=torch.complex128, device="cuda")
    factor.solve_lu_device(f, x)
    lib.rs_debug_col_times(ctypes.c_void_p(buf.data_ptr()))
    factor.solve_lu_device(f, x)
    torch.cuda.synchronize()
    lib.rs_debug_col_times(None)
    t = buf[:3 * rows].view(rows, 3).cpu().numpy()
    it = np.diff(t[:, 0])
    print(cfg, "L rows", rows, "cycles/row median", np.median(it), "mean", it.mean())
    print("  start->fetched", np.median(t[:, 1] - t[:, 0]), " fetched->synced",
          np.median(t[:, 2] - t[:, 1]), " synced->next start", np.median(t[1:, 0] - t[:-1, 2]))




def in_solver(cfg="c2"):
    """Same clocks, but for the applies inside the device-resident solver."""
    from paper_1504_06768_b200 import steady
    c = configs.CONFIGS[cfg]
    L = liouville.build_liouvillian(*c["build"]())
    sh = liouville.shift(L)
    fwd, inv = ordering.rcm_device(sh.matrix)
    A = ordering.permute(sh.matrix, fwd, inv)
    P = ordering.permute(L.matrix, fwd, inv)
    f = factor.factor_batch(A, c["d"], c["p"])
    rows = int(f.Ls[0][-1].item())
    buf = torch.zeros(3 * rows + 16, dtype=torch.int64, device="cuda")
    lib = _lib.load()
    lib.rs_debug_col_times.argtypes = [ctypes.c_void_p]
    x0 = torch.from_numpy(steady.start_vector(A.n, c["seed"])).cuda()
    lib.rs_debug_col_times(ctypes.c_void_p(buf.data_ptr()))
    steady._solve(_lib.INV_BICGSTAB, A, P, f, x0, c["tol"], 1000, 20, True)
    torch.cuda.synchronize()
    lib.rs_debug_col_times(None)
    t = buf[:3 * rows].view(rows, 3).cpu().numpy()
    it = np.diff(t[:, 0])
    print(cfg, "IN SOLVER L rows", rows, "cycles/row median", np.median(it), "mean", it.mean())
    print("  start->fetched", np.median(t[:, 1] - t[:, 0]), " fetched->synced",
          np.median(t[:, 2] - t[:, 1]), " synced->next start", np.median(t[1:, 0] - t[:-1, 2]))


if __name__ == "__main__":
    for c in sys.argv[1:] or ["c4", "c2"]:
        if c.startswith("solver:"):
            in_solver(c.split(":")[1])
        else:
            main(c)
