"""Config 5: what one BiCGStab iteration of the grid-wide solver costs, with and
without the block-Jacobi apply, against the standalone SpMV / apply launches."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1504_06768_b200 import _lib, configs, factor, liouville, ordering, sharded, steady  # noqa: E402
from bench import WORKLOADS  # noqa: E402


def ev(fn, reps=3):
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


_, bkw, skw, _ = WORKLOADS["c5"]
H, c = configs.CONFIGS[WORKLOADS["c5"][0]]["build"](**bkw)
L = liouville.build_liouvillian(H, c)
sh = liouville.shift(L)
fwd, inv = ordering.rcm_device(sh.matrix)
A = ordering.permute(sh.matrix, fwd, inv)
P = ordering.permute(L.matrix, fwd, inv)
n = A.n
M = sharded._block_jacobi((A.row_ptr, A.col_idx, A.values), 0, n, n // skw["blocks"], skw["d"],
                          skw["p"], skw["pivot_floor"], skw["early_drop"])
M.ensure_levels()
x = torch.randn(n, dtype=torch.complex128, device="cuda")
y = torch.empty_like(x)
t_spmv = ev(lambda: _lib.call("rs_csr_matvec", 1, n, _lib.ptr(A.row_ptr), _lib.ptr(A.col_idx),
                              _lib.ptr(A.values), _lib.ptr(x), _lib.ptr(y), _lib.stream_ptr()), 10)
t_apply = ev(lambda: factor.solve_lu_levels(M, x), 5)
print(f"standalone: SpMV {t_spmv:.3f} ms, apply {t_apply:.3f} ms", flush=True)
rhs = torch.from_numpy(steady.start_vector(n, 3)).cuda()
res = {}
for its in (20, 60):
    def plain():
        res["st"] = steady._solve_grid(_lib.LIN_BICGSTAB, A, None, None, rhs, 1e-300, its, 20, False)[1]

    def prec():
        res["st"] = steady._solve_grid(_lib.LIN_BICGSTAB, A, None, M, rhs, 1e-300, its, 20, False)[1]

    t0 = ev(plain, 2)
    i0 = int(res["st"]["inner_total"][0])
    t1 = ev(prec, 2)
    i1 = int(res["st"]["inner_total"][0])
    print(f"max_iter {its}: unpreconditioned {t0:.1f} ms / {i0} its = {t0 / max(i0, 1):.3f} ms/it; "
          f"block-Jacobi {t1:.1f} ms / {i1} its = {t1 / max(i1, 1):.3f} ms/it", flush=True)
