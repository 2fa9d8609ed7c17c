"""cProfile of one c4 bench step (host view: where Python blocks or works)."""
import cProfile
import os
import pstats
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1504_06768_b200 import configs, liouville, steady  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 512
L = liouville.build_liouvillian_batch([configs.jc_sweep(i) for i in range(count)])
seeds = [2 + i for i in range(count)]
kw = dict(tol=1e-12, inner="direct", ordering_name="rcm")
for _ in range(3):
    steady.inverse_power_batch(L, seeds, **kw)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(3):
    steady.inverse_power_batch(L, seeds, **kw)
    torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("cumulative").print_stats(45)
st.sort_stats("tottime").print_stats(25)
