"""solve_direct (complete LU of the trace-modified c3 Liouvillian, n=57,600,
fill ~184) and inverse_power(inner="direct") on c3 -- SURVEY 8(f) row f1."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1504_06768_b200 import configs, liouville, steady  # noqa: E402


def main():
    c = configs.CONFIGS["c3"]
    L = liouville.build_liouvillian(*c["build"]())
    t = time.perf_counter()
    r = steady.solve_direct(L, ordering_name="rcm")
    print(f"c3 solve_direct: wall {time.perf_counter() - t:.2f}s factor {r.factor_time:.2f}s "
          f"solve {r.solve_time:.3f}s fill {r.fill_factor:.1f} residual {r.residual:.2e}",
          flush=True)
    g = os.path.join(ROOT, "tests", "golden", "c3.npz")
    if os.path.exists(g):
        gd = np.load(g)
        for k in gd.files:
            if k.endswith("_rho"):
                td = 0.5 * float(np.sum(np.abs(np.linalg.eigvalsh(r.rho - gd[k]))))
                print(f"  trace distance vs reference {k}: {td:.2e}")
    t = time.perf_counter()
    r2 = steady.inverse_power(L, tol=1e-12, inner="direct", ordering_name="rcm")
    print(f"c3 inverse_power(direct): wall {time.perf_counter() - t:.2f}s factor "
          f"{r2.factor_time:.2f}s solve {r2.solve_time:.3f}s residual {r2.residual:.2e}",
          flush=True)


if __name__ == "__main__":
    main()
