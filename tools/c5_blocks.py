"""Per-block outcome of the c5 block-Jacobi ILUTP (which diagonal block hits a
zero pivot, and at which step), for comparison with the C oracle on one
extracted block.
    python tools/c5_blocks.py [N=40] [blocks=8] [d=1e-5] [p=10]"""
import ctypes
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1504_06768_b200 import _lib, configs, factor, liouville, ordering  # noqa: E402
from paper_1504_06768_b200.sparse import DeviceCSR  # noqa: E402


def main(N="40", blocks="8", d="1e-5", p="10"):
    N, blocks, d, p = int(N), int(blocks), float(d), float(p)
    t = time.perf_counter()
    L = liouville.build_liouvillian(*configs.kerr_kerr(N=N))
    S = liouville.shift(L).matrix
    fwd, inv = ordering.rcm_device(S)
    A = ordering.permute(S, fwd, inv)
    n = A.n
    block = n // blocks
    orp = torch.empty(n + 1, dtype=torch.int32, device="cuda")
    nnz = ctypes.c_int64(0)
    st = _lib.stream_ptr()
    _lib.call("rs_block_extract", n, block, 0, _lib.ptr(A.row_ptr), _lib.ptr(A.col_idx),
              _lib.ptr(A.values), _lib.ptr(orp), None, None, ctypes.byref(nnz), st)
    oci = torch.empty(nnz.value, dtype=torch.int32, device="cuda")
    ov = torch.empty(nnz.value, dtype=torch.complex128, device="cuda")
    _lib.call("rs_block_extract", n, block, 0, _lib.ptr(A.row_ptr), _lib.ptr(A.col_idx),
              _lib.ptr(A.values), _lib.ptr(orp), _lib.ptr(oci), _lib.ptr(ov),
              ctypes.byref(nnz), st)
    B = DeviceCSR(block, blocks, orp, oci, ov)
    nnz_b = B.row_ptr.diff().reshape(blocks, block).sum(1).cpu().numpy()
    print(f"N={N} n={n} blocks={blocks} nnz per block {nnz_b.tolist()} "
          f"({time.perf_counter() - t:.1f}s)", flush=True)
    f = factor.factor_batch(B, d, p, raise_on_fail=False)
    torch.cuda.synchronize()
    print(f"factor {time.perf_counter() - t:.1f}s  fail step per block {f.fail.tolist()}  "
          f"fill {np.round(f.fill_factors, 3).tolist()}", flush=True)


if __name__ == "__main__":
    main(*sys.argv[1:])
