"""c5 block-Jacobi factorization (40 blocks) vs pipeline knobs: warps per block,
frontier-poll naps."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1504_06768_b200 import configs, liouville, ordering, sharded  # noqa: E402

L = liouville.build_liouvillian(*configs.kerr_kerr(N=40))
S = liouville.shift(L)
fwd, inv = ordering.rcm_device(S.matrix)
A = ordering.permute(S.matrix, fwd, inv)
n = A.n
for knobs in ({}, {"RHOSOLVE_ILU_WARPS": "8"}, {"RHOSOLVE_ILU_WARPS": "4"}, {"RHOSOLVE_ILU_WARPS": "32"},
              {"RHOSOLVE_ILU_NAPSTEP": "16"}, {"RHOSOLVE_ILU_NAPSTEP": "256"},
              {"RHOSOLVE_ILU_HOTNAP": "32"}):
    for k in ("RHOSOLVE_ILU_WARPS", "RHOSOLVE_ILU_NAPSTEP", "RHOSOLVE_ILU_HOTNAP"):
        os.environ.pop(k, None)
    os.environ.update(knobs)
    best = 1e9
    for rep in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        M = sharded._block_jacobi((A.row_ptr, A.col_idx, A.values), 0, n, n // 40, 1e-2, 2.0, 1.0, True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    print(f"{knobs}: factor {best:.3f} s  fill {float(M.fill_factors.mean()):.3f}", flush=True)
