"""How long the main thread waits for the start vectors in a c4 step."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1504_06768_b200 import configs, liouville, steady  # noqa: E402

L = liouville.build_liouvillian_batch([configs.jc_sweep(i) for i in range(512)])
seeds = [2 + i for i in range(512)]
kw = dict(tol=1e-12, inner="direct", ordering_name="rcm")
import concurrent.futures as cf
orig = cf.Future.result
waits = []


def timed(self, timeout=None):
    t0 = time.perf_counter()
    r = orig(self, timeout)
    waits.append((time.perf_counter() - t0, type(r).__name__))
    return r


for _ in range(3):
    steady.inverse_power_batch(L, seeds, **kw)
cf.Future.result = timed
ts = []
for _ in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    steady.inverse_power_batch(L, seeds, **kw)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
print("threads", steady._DRAW_THREADS, "step ms", [round(1e3 * t, 2) for t in ts])
print("waits ms (tuple results = the main thread's x0 wait):",
      [(round(1e3 * w, 2), k) for w, k in waits if k == "tuple"])
