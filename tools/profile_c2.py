"""Profiling driver: one c2 solve's hot kernels, standalone, for ncu.

    python tools/profile_c2.py            # ILUTP, ILU apply x3, fused solver
Each kernel is launched on its own so `ncu -k regex:...` can pick it.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1504_06768_b200 import _lib, configs, factor, liouville, ordering, steady  # noqa: E402


def main(cfg="c2"):
    c = configs.CONFIGS[cfg]
    H, cops = c["build"]()
    L = liouville.build_liouvillian(H, cops)
    sh = liouville.shift(L)
    fwd, inv = ordering.rcm_device(sh.matrix)
    A = ordering.permute(sh.matrix, fwd, inv)
    P = ordering.permute(L.matrix, fwd, inv)
    f = factor.factor_batch(A, c["d"], c["p"])
    x = torch.randn(A.n, dtype=torch.complex128, device="cuda")
    for _ in range(3):
        factor.solve_lu_device(f, x)
    x0 = torch.from_numpy(steady.start_vector(A.n, c["seed"])).cuda()
    xs, st = steady._solve(_lib.INV_BICGSTAB, A, P, f, x0, c["tol"], 1000, 20, True)
    torch.cuda.synchronize()
    print("ok", st)


if __name__ == "__main__":
    main(*sys.argv[1:])
