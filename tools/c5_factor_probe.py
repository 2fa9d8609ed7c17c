"""Per-column phase timing (clock64) of block 0 in config 5's block-Jacobi ILUTP."""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1504_06768_b200 import _lib, configs, liouville, ordering, sharded  # noqa: E402

L = liouville.build_liouvillian(*configs.kerr_kerr(N=40))
S = liouville.shift(L)
fwd, inv = ordering.rcm_device(S.matrix)
A = ordering.permute(S.matrix, fwd, inv)
n = A.n
nb = n // 40
lib = _lib.load()
lib.rs_debug_factor_probe.argtypes = [ctypes.c_void_p]
buf = torch.zeros(nb * 6, dtype=torch.int64, device="cuda")
args = ((A.row_ptr, A.col_idx, A.values), 0, n, nb, 1e-2, 2.0, 1.0, True)
sharded._block_jacobi(*args)
lib.rs_debug_factor_probe(ctypes.c_void_p(buf.data_ptr()))
M = sharded._block_jacobi(*args)
torch.cuda.synchronize()
lib.rs_debug_factor_probe(None)
p = buf.view(nb, 6).cpu().numpy().astype(np.int64)
fin = p[:, 4]
gap = np.diff(fin)
ok = (gap > 0) & (gap < 1e7)
print("cycles per column: median %.0f mean %.0f" % (np.median(gap[ok]), gap[ok].mean()))
print("tail phases (median cycles): ready-after-prev %.0f  pivot+Ldrop %.0f  cap %.0f  emit+publish %.0f" % (
    np.median((p[1:, 1] - fin[:-1])[ok]), np.median(p[:, 2] - p[:, 1]), np.median(p[:, 3] - p[:, 2]),
    np.median(p[:, 4] - p[:, 3])))
print("column work start->ready median %.0f; fraction of columns ready after the previous one: %.2f" % (
    np.median(p[:, 1] - p[:, 0]), ((p[1:, 1] > fin[:-1])[ok]).mean()))
lp = M.raw[0].view(40, nb + 1)[0].cpu().numpy()
up = M.raw[3].view(40, nb + 1)[0].cpu().numpy()
print("block 0: L entries per column %.1f, U entries per column %.1f" % (lp[-1] / nb, up[-1] / nb))
