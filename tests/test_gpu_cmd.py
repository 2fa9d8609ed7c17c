"""The 'cmd' ordering on the GPU path: column-ordered
LU / ILUTP bit-identical to the reference's factors (via the pinned oracle),
and solve_direct / solve_iterative / inverse_power with ordering_name="cmd"
against the reference's steady states (tests/golden/cmd.npz)."""
import math
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_1504_06768_b200 import configs, factor, liouville, steady
from paper_1504_06768_b200.sparse import CSRMatrix, Permutation, from_host
from tests.helpers import bits_equal

pytestmark = pytest.mark.gpu
G = np.load(os.path.join(os.path.dirname(__file__), "golden", "cmd.npz"))


@pytest.mark.parametrize("name", ["c1", "c4"])
@pytest.mark.parametrize("d,p", [(0.0, math.inf), (1e-5, 10.0)])
def test_column_ordered_factors_bit_exact(cuda, name, d, p):
    rp = G[f"lu_{name}_rp"]
    n = len(rp) - 1
    host = CSRMatrix(n, n, rp, G[f"lu_{name}_ci"], G[f"lu_{name}_v"])
    colp = Permutation(G[f"lu_{name}_colfwd"])
    A = from_host(host)
    f = factor.lu(A, colp) if d == 0.0 else factor.ilutp(A, d, p, colp)
    fo = O.factorize_raw(O.CSR(n, n, host.row_ptr, host.col_idx, host.values), d, p,
                         q=colp.inverse)
    lp, li, lx, up, ui, ux, pinv = f.system_raw(0)
    assert bits_equal(lp, fo.Lp) and bits_equal(li, fo.Li) and bits_equal(lx, fo.Lx)
    assert bits_equal(up, fo.Up) and bits_equal(ui, fo.Ui) and bits_equal(ux, fo.Ux)
    assert bits_equal(pinv, fo.pinv)
    assert np.array_equal(f.col_perm.forward, colp.forward)
    # solve_lu scatters x[q] = y (factor.py:147-148)
    b = np.random.default_rng(3).standard_normal(n) + 0.25j
    y = fo.solve(b)
    x = np.empty_like(y)
    x[colp.inverse] = y
    assert bits_equal(factor.solve_lu(f, b), x)


def _L(name):
    H, c = configs.kerr() if name == "c1" else configs.jc_sweep(7)
    return liouville.build_liouvillian(H, c)


RUNS = {
    "direct": lambda L: steady.solve_direct(L, "cmd"),
    "bicgstab": lambda L: steady.solve_iterative(L, "cmd", "bicgstab", d=1e-5, p=10.0, tol=1e-12),
    "power": lambda L: steady.inverse_power(L, tol=1e-12, inner="direct", ordering_name="cmd",
                                            seed=0),
    "power_bicgstab": lambda L: steady.inverse_power(L, tol=1e-12, inner="iterative",
                                                     ordering_name="cmd", solver="bicgstab",
                                                     d=1e-4, p=300.0, seed=0),
}


@pytest.mark.parametrize("name", ["c1", "c4"])
@pytest.mark.parametrize("key", list(RUNS))
def test_cmd_steady_states_match_reference(cuda, name, key):
    L = _L(name)
    err = f"{name}_{key}_error"
    if err in G.files:
        exc = {"PowerIterationError": steady.PowerIterationError,
               "InnerSolverError": steady.InnerSolverError}.get(str(G[err]), Exception)
        with pytest.raises((exc, factor.PreconditionerBreakdownError)):
            RUNS[key](L)
        return
    r = RUNS[key](L)
    assert r.ordering == str(G[f"{name}_{key}_label"])
    assert r.residual <= 1e-10
    assert O.trace_distance(r.rho, G[f"{name}_{key}_rho"]) <= 1e-6
