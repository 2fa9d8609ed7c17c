"""c5 block-Jacobi factorization time vs CTAs per block (RHOSOLVE_ILU_CPS).
    python tools/c5_factor.py N blocks d p"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1504_06768_b200 import configs, liouville, ordering, sharded  # noqa: E402


def main(N="40", blocks="16", d="1e-2", p="2"):
    N, blocks, d, p = int(N), int(blocks), float(d), float(p)
    L = liouville.build_liouvillian(*configs.kerr_kerr(N=N))
    S = liouville.shift(L)
    fwd, inv = ordering.rcm_device(S.matrix)
    A = ordering.permute(S.matrix, fwd, inv)
    n = A.n
    for cps in os.environ.get("CPS_LIST", "9,4,2,1").split(","):
        os.environ["RHOSOLVE_ILU_CPS"] = cps
        for rep in range(2):
            torch.cuda.synchronize()
            t = time.perf_counter()
            M = sharded._block_jacobi((A.row_ptr, A.col_idx, A.values), 0, n, n // blocks, d, p,
                                      1.0, True)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t
        print(f"N={N} blocks={blocks} cps={cps}: factor {dt:.3f}s fill {float(M.fill_factors.mean()):.3f}",
              flush=True)


if __name__ == "__main__":
    main(*sys.argv[1:])
