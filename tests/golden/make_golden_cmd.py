"""Golden fixtures for the 'cmd' ordering row, written
by the REFERENCE rhosolve: tests/golden/cmd.npz holds
  * weighted_mbm forward maps and col_min_degree orders on a seeded random
    corpus (dense-ish and sparse, integer-valued entries for magnitude ties,
    some structurally singular) and on the c1 / c4 (Delta_c index 7)
    shifted, modified and plain Liouvillians;
  * rho from solve_direct / solve_iterative / inverse_power with
    ordering_name="cmd" on c1 and the c4 instance, plus each result's
    ordering label.
Run in the build container: python tests/golden/make_golden_cmd.py
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
for cand in (os.path.join(ROOT, "oracle", "_ref"), "/root/reference/pkg/src"):
    if os.path.isdir(os.path.join(cand, "rhosolve")):
        sys.path.insert(0, cand)
        break

from rhosolve import liouville as RL  # noqa: E402
from rhosolve import operators as RO  # noqa: E402
from rhosolve import ordering as ROrd  # noqa: E402
from rhosolve import sparse as RS  # noqa: E402
from rhosolve import steady as RSt  # noqa: E402

from paper_1504_06768_b200 import configs  # noqa: E402


def corpus():
    rng = np.random.default_rng(2024)
    out = []
    for t in range(60):
        n = int(rng.integers(2, 45))
        dens = rng.uniform(0.04, 0.45)
        mask = rng.random((n, n)) < dens
        if t % 4 != 3:
            mask[np.arange(n), rng.permutation(n)] = True  # mostly nonsingular
        r, c = np.nonzero(mask)
        v = rng.standard_normal(len(r)) + 1j * rng.standard_normal(len(r))
        if t % 3 == 0:
            v = np.round(2 * v) / 2  # magnitude ties, some exact zeros
        out.append(RS.SparseComplexMatrix.from_coo(n, n, r, c, v, prune=False))
    return out


def main():
    res = {}
    mats = corpus()
    H1, c1 = configs.kerr(ops=RO)
    H4, c4 = configs.jc_sweep(7, ops=RO)
    for name, (H, c) in (("c1", (H1, c1)), ("c4", (H4, c4))):
        L = RL.build_liouvillian(H, c)
        mats += [L.matrix, RL.shift(L).matrix, RL.build_modified(L).matrix]
    for k, m in enumerate(mats):
        res[f"m{k}_rp"], res[f"m{k}_ci"], res[f"m{k}_v"] = m.row_ptr, m.col_idx, m.values
        try:
            res[f"m{k}_mbm"] = ROrd.weighted_mbm(m).forward
        except ROrd.StructurallySingularError:
            res[f"m{k}_mbm"] = np.array([-1])
        res[f"m{k}_cmd"] = ROrd.col_min_degree(m).inverse  # the elimination order
    res["count"] = np.array(len(mats))
    # factorization with the cmd column order: the reference's raw factors
    from rhosolve import factor as RF
    import hashlib
    for name, (H, c) in (("c1", (H1, c1)), ("c4", (H4, c4))):
        L = RL.build_liouvillian(H, c)
        m, _, _, _, colp, _ = RSt._prepare(RL.build_modified(L), "cmd")
        res[f"lu_{name}_rp"], res[f"lu_{name}_ci"], res[f"lu_{name}_v"] = (
            m.row_ptr, m.col_idx, m.values)
        res[f"lu_{name}_colfwd"] = colp.forward
        for tag, f in (("lu", RF.lu(m, colp)), ("ilu", RF.ilutp(m, 1e-5, 10.0, colp))):
            h = hashlib.sha256()
            for a in (f._Lp, f._Li, f._Lx, f._Up, f._Ui, f._Ux, f.row_perm.forward):
                h.update(np.ascontiguousarray(a).tobytes())
            res[f"lu_{name}_{tag}_sha"] = np.array(h.hexdigest())
    for name, (H, c) in (("c1", (H1, c1)), ("c4", (H4, c4))):
        L = RL.build_liouvillian(H, c)
        runs = {
            "direct": lambda: RSt.solve_direct(L, "cmd"),
            "bicgstab": lambda: RSt.solve_iterative(L, "cmd", "bicgstab", d=1e-5, p=10.0,
                                                    tol=1e-12),
            "power": lambda: RSt.inverse_power(L, tol=1e-12, inner="direct",
                                               ordering_name="cmd", seed=0),
            "power_bicgstab": lambda: RSt.inverse_power(L, tol=1e-12, inner="iterative",
                                                        ordering_name="cmd", solver="bicgstab",
                                                        d=1e-4, p=300.0, seed=0),
        }
        for key, fn in runs.items():
            try:
                r = fn()
                res[f"{name}_{key}_rho"] = r.rho
                res[f"{name}_{key}_label"] = np.array(r.ordering)
                res[f"{name}_{key}_residual"] = np.array(r.residual)
            except Exception as e:  # noqa: BLE001 -- record the reference's failure
                res[f"{name}_{key}_error"] = np.array(type(e).__name__)
    np.savez_compressed(os.path.join(HERE, "cmd.npz"), **res)
    print(sorted(k for k in res if not k.startswith("m")))


if __name__ == "__main__":
    main()
