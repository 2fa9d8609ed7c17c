"""Config 5: factorization time and fill of every block-Jacobi block on its own."""
import ctypes
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1504_06768_b200 import _lib, configs, factor, liouville, ordering, sharded  # noqa: E402
from paper_1504_06768_b200.sparse import DeviceCSR  # noqa: E402

L = liouville.build_liouvillian(*configs.kerr_kerr(N=40))
S = liouville.shift(L)
fwd, inv = ordering.rcm_device(S.matrix)
A = ordering.permute(S.matrix, fwd, inv)
n = A.n
nb = n // 40
M = sharded._block_jacobi((A.row_ptr, A.col_idx, A.values), 0, n, nb, 1e-2, 2.0, 1.0, True)
lnnz, unnz = M.lnnz, M.unnz
rp = A.row_ptr.cpu().numpy()
times = []
for b in range(40):
    # rows [b*nb, (b+1)*nb) restricted to their diagonal block, as one system
    t0 = time.perf_counter()
    Mb = sharded._block_jacobi((A.row_ptr[b * nb:(b + 1) * nb + 1] - A.row_ptr[b * nb],
                                A.col_idx[rp[b * nb]:rp[(b + 1) * nb]],
                                A.values[rp[b * nb]:rp[(b + 1) * nb]]), b * nb, nb, nb, 1e-2, 2.0, 1.0, True)
    torch.cuda.synchronize()
    times.append(time.perf_counter() - t0)
times = np.array(times)
print("per-block factor time (s), alone on the GPU:")
print(np.round(times, 3).tolist())
print("L+U entries per block (k):", np.round((lnnz + unnz) / 1e3).astype(int).tolist())
print(f"max {times.max():.3f} mean {times.mean():.3f} sum {times.sum():.2f}")
