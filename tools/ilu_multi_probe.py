"""Multi-CTA factorization of the large single systems (c3 ILUTP(1e-4,300))
and the c5 N=20 block-Jacobi blocks vs the single-CTA kernel: timing and
bit-identity of the factors (tuning)."""
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1504_06768_b200 import configs, factor, liouville, ordering  # noqa: E402


def run(A, d, p, label):
    out = {}
    for cps in os.environ.get("CPS_LIST", "1,4,8,16").split(","):
        os.environ["RHOSOLVE_ILU_CPS"] = cps
        torch.cuda.synchronize()
        t = time.perf_counter()
        f = factor.factor_batch(A, d, p)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        import numpy as np
        raw = [np.asarray(x) for b in range(f.nsys) for x in f.system_raw(b)]
        out[cps] = raw
        same = all(a.shape == b.shape and np.array_equal(a.view(np.int64) if a.dtype.kind == "c"
                                                          else a,
                                                          b.view(np.int64) if b.dtype.kind == "c"
                                                          else b)
                   for a, b in zip(raw, next(iter(out.values()))))
        print(f"{label} cps={cps}: factor {dt:.3f}s fill {float(f.fill_factors.mean()):.2f} "
              f"{'bit-identical to the first run' if same else 'MISMATCH'}", flush=True)


def main():
    for name in ("c2", "c1"):
        cc = configs.CONFIGS[name]
        Lc = liouville.build_liouvillian(*cc["build"]())
        shc = liouville.shift(Lc)
        fc, ic = ordering.rcm_device(shc.matrix)
        run(ordering.permute(shc.matrix, fc, ic), cc["d"], cc["p"], f"{name} ILUTP")
    if os.environ.get("ONLY_SMALL"):
        return
    c = configs.CONFIGS["c3"]
    L = liouville.build_liouvillian(*c["build"]())
    sh = liouville.shift(L)
    fwd, inv = ordering.rcm_device(sh.matrix)
    A = ordering.permute(sh.matrix, fwd, inv)
    run(A, c["d"], c["p"], "c3 ILUTP(1e-4,300)")
    # c5 N=20 block-Jacobi blocks: 8 diagonal blocks of 20,000 rows
    import ctypes
    from paper_1504_06768_b200 import _lib
    from paper_1504_06768_b200.sparse import DeviceCSR
    H, cops = configs.kerr_kerr(N=20)
    L5 = liouville.build_liouvillian(H, cops)
    s5 = liouville.shift(L5)
    f5, i5 = ordering.rcm_device(s5.matrix)
    A5 = ordering.permute(s5.matrix, f5, i5)
    n, block = A5.n, A5.n // 8
    orp = torch.empty(n + 1, dtype=torch.int32, device="cuda")
    nnz = ctypes.c_int64(0)
    args = lambda oc, ov: (n, block, 0, _lib.ptr(A5.row_ptr), _lib.ptr(A5.col_idx),  # noqa: E731
                           _lib.ptr(A5.values), _lib.ptr(orp), oc, ov, ctypes.byref(nnz),
                           _lib.stream_ptr())
    _lib.call("rs_block_extract", *args(None, None))
    oci = torch.empty(nnz.value, dtype=torch.int32, device="cuda")
    ov = torch.empty(nnz.value, dtype=torch.complex128, device="cuda")
    _lib.call("rs_block_extract", *args(_lib.ptr(oci), _lib.ptr(ov)))
    run(DeviceCSR(block, 8, orp, oci, ov), 1e-5, 10.0, "c5 N=20 8 blocks ILUTP(1e-5,10)")


if __name__ == "__main__":
    main()
