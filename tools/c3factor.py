import os, sys, time
sys.path.insert(0, '/root/repo')
import torch
from paper_1504_06768_b200 import configs, factor, liouville, ordering
c = configs.CONFIGS["c3"]
L = liouville.build_liouvillian(*c["build"]())
sh = liouville.shift(L)
fwd, inv = ordering.rcm_device(sh.matrix)
A = ordering.permute(sh.matrix, fwd, inv)
for rep in range(2):
    torch.cuda.synchronize(); t = time.perf_counter()
    f = factor.factor_batch(A, c["d"], c["p"])
    torch.cuda.synchronize()
    print(os.environ.get("RHOSOLVE_B200_LIB", "current"), "c3 factor s", time.perf_counter() - t, flush=True)
