"""One steady-state solve of a BASELINE config through the public API
(for ncu captures of the solver kernel)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1504_06768_b200 import configs, liouville, steady  # noqa: E402


def main(cfg="c2", csc="1"):
    c = configs.CONFIGS[cfg]
    L = liouville.build_liouvillian(*c["build"]())
    kw = dict(tol=c["tol"], inner="iterative", ordering_name="rcm", solver="bicgstab",
              d=c["d"], p=c["p"], seed=c["seed"])
    if csc == "0":
        from paper_1504_06768_b200 import _lib
        orig = _lib.load().rs_col_sweep_supported
        _lib.load().rs_col_sweep_supported = lambda n: 0
    r = steady.inverse_power(L, **kw)
    torch.cuda.synchronize()
    print(cfg, "csc" if csc != "0" else "rows", "solve_time", r.solve_time, "inner", r.inner_iterations,
          "residual", r.residual)


if __name__ == "__main__":
    main(*sys.argv[1:])
