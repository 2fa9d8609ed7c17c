import os, sys, time
sys.path.insert(0, '/root/repo')
import torch, numpy as np
from paper_1504_06768_b200 import _lib, configs, factor, liouville, ordering, steady
c = configs.CONFIGS["c2"]
L = liouville.build_liouvillian(*c["build"]())
sh = liouville.shift(L)
fwd, inv = ordering.rcm_device(sh.matrix)
A = ordering.permute(sh.matrix, fwd, inv)
P = ordering.permute(L.matrix, fwd, inv)
f = factor.factor_batch(A, c["d"], c["p"])
x0 = torch.from_numpy(steady.start_vector(A.n, 1)).cuda()
for threads in (288, 512, 160, 512):
    for rep in range(2):
        torch.cuda.synchronize(); t = time.perf_counter()
        x, st = steady._solve(_lib.INV_BICGSTAB, A, P, f, x0, 1e-12, 1000, 20, True, threads)
        torch.cuda.synchronize()
    print(threads, "solver ms", 1e3 * (time.perf_counter() - t), st["inner_total"])
xx = torch.randn(A.n, dtype=torch.complex128, device="cuda")
for rep in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(20): factor.solve_lu_device(f, xx)
    torch.cuda.synchronize()
print("20 standalone applies ms", 1e3 * (time.perf_counter() - t))
import ctypes
lib = _lib.load()
lib.rs_debug_solver_prof.argtypes = [ctypes.c_void_p]
pf = torch.zeros(4, dtype=torch.int64, device="cuda")
lib.rs_debug_solver_prof(ctypes.c_void_p(pf.data_ptr()))
torch.cuda.synchronize(); t = time.perf_counter()
x, st = steady._solve(_lib.INV_BICGSTAB, A, P, f, x0, 1e-12, 1000, 20, True, 512)
torch.cuda.synchronize()
lib.rs_debug_solver_prof(None)
tot = (time.perf_counter() - t) * 1.965e9
p = pf.cpu().numpy()
print("total cycles", tot, "psolve cycles", p[0], "calls", p[1], "spmv cycles", p[2])
