"""Multi-consumer column sweeps (colsweep.cuh col_consume_multi): bit-exact
against the oracle for 1, 2, 4 consumer warps, and the config-3 apply time."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1504_06768_b200 import configs, factor, liouville, ordering  # noqa: E402
from paper_1504_06768_b200.sparse import CSRMatrix, from_host  # noqa: E402
from tools.time_grid import ev_time  # noqa: E402


def check(name, m, d, p):
    fo = O.factorize_raw(m, d, p)
    f = factor.factor_batch(from_host(CSRMatrix(m.n, m.m, m.rp, m.ci, m.v)), d, p)
    rng = np.random.default_rng(1)
    b = rng.standard_normal(m.n) + 1j * rng.standard_normal(m.n)
    ref = fo.solve(b)
    for w in ("1", "2", "4"):
        os.environ["RHOSOLVE_COL_CONSUMERS"] = w
        x = factor.solve_lu(f, b)
        ok = np.array_equal(x.view(np.float64), ref.view(np.float64))
        print(f"{name} consumers={w}: bit-exact {ok}", flush=True)
        assert ok


def main():
    os.environ["RHOSOLVE_GRID_MIN_N"] = "100000000"
    for name, (H, c), D in (("c1", configs.kerr(), 20), ("c2", configs.jc_rwa(), 80)):
        Lo = O.build_liouvillian(H.matrix, [x.matrix for x in c])
        for variant, m in (("shift", O.shift(Lo)), ("mod", O.build_modified(Lo, D)[0])):
            fwd, _ = O.rcm(m)
            pm = O.permute(m, fwd)
            check(f"{name} {variant} lu", pm, 0.0, float("inf"))
            if variant == "mod":
                check(f"{name} {variant} ilutp", pm, 1e-5, 10.0)
    # config 3: time the apply for 1 / 2 / 4 / 6 consumers
    L = liouville.build_liouvillian(*configs.optomech())
    S = liouville.shift(L)
    fwd, inv = ordering.rcm_device(S.matrix)
    A = ordering.permute(S.matrix, fwd, inv)
    f = factor.factor_batch(A, 1e-4, 300.0)
    b = torch.randn(A.n, dtype=torch.complex128, device="cuda")
    base = None
    f.ensure_cols()
    print(f"c3 factor reach {f.reach}", flush=True)
    for win in ("0", "1"):
        os.environ["RHOSOLVE_COL_WINDOW"] = win
        for w in ("1", "2", "4", "6"):
            os.environ["RHOSOLVE_COL_CONSUMERS"] = w
            ms = ev_time(lambda: factor.solve_lu_device(f, b), reps=3)
            x = factor.solve_lu_device(f, b).cpu().numpy()
            if base is None:
                base = x
            same = np.array_equal(x.view(np.float64), base.view(np.float64))
            print(f"c3 apply window={win} consumers={w}: {ms:.2f} ms, equal to the 1-consumer "
                  f"global sweep: {same}", flush=True)
    del os.environ["RHOSOLVE_COL_CONSUMERS"], os.environ["RHOSOLVE_COL_WINDOW"]
    ms = ev_time(lambda: factor.solve_lu_device(f, b), reps=3)
    print(f"c3 apply defaults: {ms:.2f} ms", flush=True)


if __name__ == "__main__":
    main()
