"""'cmd' ordering: the host-native weighted MBM and
column minimum degree (csrc/cmd_order.cu) against the reference's own
permutations (tests/golden/cmd.npz, made by tests/golden/make_golden_cmd.py),
and the oracle's column-ordered factorization against the reference's
factors.  Host code only: runs without a GPU."""
import hashlib
import math
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_1504_06768_b200 import ordering
from paper_1504_06768_b200.sparse import CSRMatrix

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "cmd.npz"))


def _mat(k):
    rp = G[f"m{k}_rp"]
    n = len(rp) - 1
    return CSRMatrix(n, n, rp, G[f"m{k}_ci"], G[f"m{k}_v"])


@pytest.mark.parametrize("k", range(int(G["count"])))
def test_weighted_mbm_and_min_degree_match_reference(k):
    m = _mat(k)
    want = G[f"m{k}_mbm"]
    if want.size == 1 and want[0] == -1 and m.nrows > 1:
        with pytest.raises(ordering.StructurallySingularError):
            ordering.weighted_mbm(m)
    else:
        p = ordering.weighted_mbm(m)
        assert np.array_equal(p.forward, want)
        # a zero-free structural diagonal after the row permutation
        rows = p.forward[m.row_ids()]
        assert np.all(np.isin(np.arange(m.nrows), rows[rows == m.col_idx]))
    assert np.array_equal(ordering.col_min_degree(m).inverse, G[f"m{k}_cmd"])


def test_square_required():
    m = CSRMatrix(2, 3, [0, 1, 2], [0, 2], [1.0, 2.0])
    with pytest.raises(ValueError, match="square"):
        ordering.weighted_mbm(m)
    with pytest.raises(ValueError, match="square"):
        ordering.col_min_degree(m)


@pytest.mark.parametrize("name", ["c1", "c4"])
@pytest.mark.parametrize("tag,d,p", [("lu", 0.0, math.inf), ("ilu", 1e-5, 10.0)])
def test_oracle_column_ordered_factors_pinned(name, tag, d, p):
    rp = G[f"lu_{name}_rp"]
    n = len(rp) - 1
    A = O.CSR(n, n, rp, G[f"lu_{name}_ci"], G[f"lu_{name}_v"])
    q = np.argsort(G[f"lu_{name}_colfwd"])  # col_perm.inverse
    f = O.factorize_raw(A, d, p, q=q)
    h = hashlib.sha256()
    for a in (f.Lp, f.Li, f.Lx, f.Up, f.Ui, f.Ux, f.pinv):
        h.update(np.ascontiguousarray(a).tobytes())
    assert h.hexdigest() == str(G[f"lu_{name}_{tag}_sha"])
