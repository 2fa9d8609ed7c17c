"""Time one block-Jacobi apply and one sharded SpMV for a Kerr x Kerr size."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1504_06768_b200 import configs, factor, liouville, ordering, sharded  # noqa: E402


def main(N="20", blocks="8"):
    N, blocks = int(N), int(blocks)
    L = liouville.build_liouvillian(*configs.kerr_kerr(N=N))
    t = time.perf_counter()
    sh = liouville.shift(L)
    fwd, inv = ordering.rcm_device(sh.matrix)
    torch.cuda.synchronize()
    print(f"N={N} n={L.n}: shift+rcm {time.perf_counter() - t:.2f}s", flush=True)
    S = ordering.permute(sh.matrix, fwd, inv)
    n = S.n
    comm = sharded.Comm()
    A = sharded.ShardedMatrix(n, S.row_ptr, S.col_idx, S.values, 0, n, comm, S.values.device)
    t = time.perf_counter()
    M = sharded._block_jacobi((S.row_ptr, S.col_idx, S.values), 0, n, n // blocks, 1e-5, 10.0)
    torch.cuda.synchronize()
    print(f"factor {blocks} blocks: {time.perf_counter() - t:.2f}s", flush=True)
    ops = sharded.GpuOps(comm)
    x = torch.randn(n, dtype=torch.complex128, device="cuda")
    for name, fn in (("spmv", lambda: ops.matvec(A, x)), ("apply", lambda: ops.psolve(M, x))):
        fn()
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        print(f"{name}: {(time.perf_counter() - t) / 3 * 1e3:.2f} ms", flush=True)


if __name__ == "__main__":
    main(*sys.argv[1:])
