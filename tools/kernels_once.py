"""Launch the c4-batch SpMV and preconditioner apply once each (for ncu)."""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1504_06768_b200 import _lib, configs, factor, liouville, ordering  # noqa: E402


def main(count="512"):
    L = liouville.build_liouvillian_batch([configs.jc_sweep(i) for i in range(int(count))])
    sh = liouville.shift(L)
    fwd, inv = ordering.rcm_device(sh.matrix)
    A = ordering.permute(sh.matrix, fwd, inv)
    f = factor.factor_batch(A, 0.0, math.inf)
    x = torch.randn(A.n * A.nsys, dtype=torch.complex128, device="cuda")
    y = torch.empty_like(x)
    torch.cuda.synchronize()
    _lib.call("rs_csr_matvec", A.nsys, A.n, _lib.ptr(A.row_ptr), _lib.ptr(A.col_idx),
              _lib.ptr(A.values), _lib.ptr(x), _lib.ptr(y), _lib.stream_ptr())
    factor.solve_lu_device(f, x)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main(*sys.argv[1:])
