"""Synthetic banded unit-lower triangles through the real warp-per-row sweep:
row r has k entries at columns r-1..r-k (so every row depends on the previous
one): cycles/row vs k separates the hop cost from the per-entry cost."""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1504_06768_b200 import _lib  # noqa: E402


def main():
    lib = _lib.load()
    fn = lib.rs_debug_tri_probe
    fn.argtypes = [ctypes.c_int] + [ctypes.c_void_p] * 6 + [ctypes.c_int] * 4 + [ctypes.c_void_p]
    n = 6400
    for k in (1, 2, 4, 8, 16, 32, 64, 96):
        rows, cols = [], []
        for r in range(n):
            for j in range(min(k, r), 0, -1):
                rows.append(r)
                cols.append(r - j)
        rows, cols = np.array(rows), np.array(cols)
        rp = np.zeros(n + 1, np.int32)
        np.add.at(rp, rows + 1, 1)
        rp = np.cumsum(rp).astype(np.int32)
        vals = (0.5 / k) * np.ones(len(cols), complex)
        d_rp = torch.from_numpy(rp).cuda()
        d_ci = torch.from_numpy(cols.astype(np.int32)).cuda()
        d_v = torch.from_numpy(vals).cuda()
        x = torch.ones(n, dtype=torch.complex128, device="cuda")
        out = torch.empty_like(x)
        for threads, variant in ((256, 1), (256, 2), (512, 2), (1024, 2)):
            ts = []
            for rep in range(3):
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record()
                fn(n, d_rp.data_ptr(), d_ci.data_ptr(), d_v.data_ptr(), x.data_ptr(),
                   x.data_ptr(), out.data_ptr(), 0, variant, 1, threads, None)
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            print(f"k={k:3d} threads={threads} variant={variant}: {1e6 * min(ts) / n * 1.965:7.0f} cycles/row",
                  flush=True)


if __name__ == "__main__":
    main()
