"""Dependency-hop latency of the level-ordered sweeps: a bidiagonal system is
one chain (every row waits on the previous one), so sweep time / n is the
publish -> dependent-publish latency.  python tools/hop_probe.py [n] [band]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1504_06768_b200 import factor  # noqa: E402
from paper_1504_06768_b200.sparse import CSRMatrix, from_host  # noqa: E402
from tools.time_grid import ev_time  # noqa: E402


def main(n="20000", band="1"):
    n, band = int(n), int(band)
    rows, cols, vals = [], [], []
    for i in range(n):
        for j in range(max(0, i - band), i + 1):
            rows.append(i)
            cols.append(j)
            vals.append(4.0 + 0j if i == j else -0.5 + 0.1j)
    rp = np.zeros(n + 1, dtype=np.int64)
    np.add.at(rp, np.asarray(rows) + 1, 1)
    rp = np.cumsum(rp)
    A = from_host(CSRMatrix(n, n, rp, np.asarray(cols, dtype=np.int64),
                            np.asarray(vals, dtype=np.complex128)))
    f = factor.factor_batch(A, 0.0, float("inf"))
    f.ensure_levels()
    b = torch.randn(n, dtype=torch.complex128, device="cuda")
    for apw in (1, 2, 4, 16):
        f.Llev.apw = f.Ulev.apw = apw
        ms = ev_time(lambda: factor.solve_lu_levels(f, b), reps=3)
        print(f"n={n} band={band} L levels {f.Llev.nlevels} (G={f.Llev.G}) U levels {f.Ulev.nlevels} "
              f"apw={apw}: apply {ms:.3f} ms -> {ms * 1e6 / f.Llev.nlevels:.0f} ns per L hop")


if __name__ == "__main__":
    main(*sys.argv[1:])
