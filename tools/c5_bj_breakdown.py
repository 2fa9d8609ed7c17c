"""Config 5: where sharded._block_jacobi (the 'factor' stage) spends its time."""
import collections
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1504_06768_b200 import _lib, configs, liouville, ordering, sharded  # noqa: E402

L = liouville.build_liouvillian(*configs.kerr_kerr(N=40))
S = liouville.shift(L)
fwd, inv = ordering.rcm_device(S.matrix)
A = ordering.permute(S.matrix, fwd, inv)
n = A.n
args = ((A.row_ptr, A.col_idx, A.values), 0, n, n // 40, 1e-2, 2.0, 1.0, True)
sharded._block_jacobi(*args)
acc = collections.OrderedDict()
orig = _lib.call


def timed_call(name, *a):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = orig(name, *a)
    torch.cuda.synchronize()
    acc[name] = acc.get(name, 0.0) + time.perf_counter() - t0
    return r


_lib.call = timed_call
torch.cuda.synchronize()
t0 = time.perf_counter()
M = sharded._block_jacobi(*args)
torch.cuda.synchronize()
tot = time.perf_counter() - t0
_lib.call = orig
print(f"_block_jacobi {1e3 * tot:.1f} ms")
for k, v in acc.items():
    print(f"   {k:28s} {1e3 * v:8.2f} ms")
print(f"   torch + Python: {1e3 * (tot - sum(acc.values())):.1f} ms")
