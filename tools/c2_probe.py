"""c2 (n = 6400) doubly-iterative solve: stage times vs tuning knobs."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1504_06768_b200 import configs, liouville, steady  # noqa: E402

L = liouville.build_liouvillian(*configs.jc_rwa())
for knobs in ({}, {"RHOSOLVE_COL_CONSUMERS": "2"}, {"RHOSOLVE_COL_CONSUMERS": "3"},
              {"RHOSOLVE_COL_CONSUMERS": "4"}, {"RHOSOLVE_ILU_CPS": "4"},
              {"RHOSOLVE_ILU_CPS": "8"}, {"RHOSOLVE_ILU_CPS": "16"},
              {"RHOSOLVE_ILU_CPS": "32"}):
    for k in ("RHOSOLVE_COL_CONSUMERS", "RHOSOLVE_ILU_CPS"):
        os.environ.pop(k, None)
    os.environ.update(knobs)
    best = None
    for rep in range(4):
        r = steady.inverse_power(L, tol=1e-12, inner="iterative", ordering_name="rcm",
                                 solver="bicgstab", d=1e-4, p=300.0, seed=1)
        t = (r.build_time, r.factor_time, r.solve_time)
        best = t if best is None or sum(t) < sum(best) else best
    print(f"{knobs}: build {best[0] * 1e3:.1f} factor {best[1] * 1e3:.1f} solve {best[2] * 1e3:.1f} ms "
          f"residual {r.residual:.1e} inner {r.inner_iterations}", flush=True)
