"""Wall time of one steady-state solve per BASELINE config through the public
API (c1, c2, c3 single systems), with the stage split the API reports."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1504_06768_b200 import configs, liouville, steady  # noqa: E402


def main(names=("c1", "c2", "c3")):
    for name in names:
        c = configs.CONFIGS[name]
        L = liouville.build_liouvillian(*c["build"]())
        solver = "gmres" if name == "c3-gmres" else "bicgstab"
        kw = dict(tol=c["tol"], inner="iterative", ordering_name="rcm", solver=solver,
                  d=c["d"], p=c["p"], seed=c["seed"])
        for rep in range(2 if name != "c3" else 1):
            torch.cuda.synchronize()
            t = time.perf_counter()
            r = steady.inverse_power(L, **kw)
            wall = time.perf_counter() - t
        print(f"{name}: wall {wall:.3f}s build {r.build_time:.3f} factor {r.factor_time:.3f} "
              f"solve {r.solve_time:.3f} outer {r.iterations} inner {r.inner_iterations} "
              f"residual {r.residual:.2e} fill {r.fill_factor:.2f}", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ("c1", "c2", "c3"))
