"""The host operator algebra (paper_1504_06768_b200.sparse / .operators) builds
bit-identical operators to the reference's own modules: every BASELINE
configuration's H and collapse operators, and random complex matrices through
kron / add / matmul / transpose / adjoint.  Needs the built reference
(oracle/_ref); the committed goldens (tests/test_host.py) cover c1/c2/c4
without it."""
import os
import sys

import numpy as np
import pytest

from paper_1504_06768_b200 import configs, sparse as MS

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref")
pytestmark = pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "rhosolve")),
                                reason="oracle/_ref (the built reference) is not present")


@pytest.fixture(scope="module")
def ref():
    sys.path.insert(0, REF)
    try:
        from rhosolve import operators, sparse
    finally:
        sys.path.remove(REF)
    return operators, sparse


def same(a, b):
    return (np.array_equal(a.row_ptr, b.row_ptr) and np.array_equal(a.col_idx, b.col_idx)
            and np.array_equal(a.values.view(np.float64), b.values.view(np.float64)))


@pytest.mark.parametrize("build,kw", [
    (configs.kerr, {}), (configs.jc_rwa, {}), (configs.optomech, {}),
    (configs.kerr_kerr, {"N": 12}), (lambda **k: configs.jc_sweep(300, **k), {})])
def test_config_operators_match_reference(ref, build, kw):
    RO, _ = ref
    H1, c1 = build(ops=RO, **kw)
    H2, c2 = build(**kw)
    assert H1.dims == H2.dims and same(H1.matrix, H2.matrix)
    assert len(c1) == len(c2)
    for x, y in zip(c1, c2):
        assert same(x.matrix, y.matrix)


def test_random_complex_algebra_matches_reference(ref):
    _, RS = ref
    rng = np.random.default_rng(0)

    def pair(r, c):
        rr, cc = np.nonzero(rng.random((r, c)) < 0.5)
        v = rng.standard_normal(len(rr)) + 1j * rng.standard_normal(len(rr))
        return (RS.SparseComplexMatrix.from_coo(r, c, rr, cc, v),
                MS.CSRMatrix.from_coo(r, c, rr, cc, v))

    for _ in range(25):
        n, m = int(rng.integers(1, 9)), int(rng.integers(1, 9))
        a1, a2 = pair(n, m)
        b1, b2 = pair(m, n)
        c1, c2 = pair(n, m)
        assert same(RS.matmul(a1, b1), MS.matmul(a2, b2))
        assert same(RS.add(a1, c1, 0.5 - 1j, 2.0), MS.add(a2, c2, 0.5 - 1j, 2.0))
        assert same(RS.add(a1, a1, 1.0, -1.0), MS.add(a2, a2, 1.0, -1.0))  # all cancel
        assert same(RS.kron(a1, b1), MS.kron(a2, b2))
        assert same(RS.transpose(a1), MS.transpose(a2))
        assert same(RS.adjoint(a1), MS.adjoint(a2))
    assert same(RS.identity(5), MS.identity(5))


def test_spin_and_scalar_ops(ref):
    RO, _ = ref
    from paper_1504_06768_b200 import operators as MO
    s1, s2 = RO.spin_ops(), MO.spin_ops()
    assert set(s1) == set(s2)
    for k in s1:
        assert same(s1[k].matrix, s2[k].matrix), k
    a1, a2 = RO.destroy(7), MO.destroy(7)
    for f in (0.0, -1.0, 2.5, 1j, 0.3 - 0.2j):
        assert same((f * a1).matrix, (f * a2).matrix)
        assert same((a1 * f).matrix, (a2 * f).matrix)
    assert same((-a1).matrix, (-a2).matrix)
    assert same((a1 - a1.adjoint()).matrix, (a2 - a2.adjoint()).matrix)
    e1 = RO.embed(a1, (3, 7, 2), 1)
    e2 = MO.embed(a2, (3, 7, 2), 1)
    assert e1.dims == e2.dims and same(e1.matrix, e2.matrix)
    assert same(RO.identity_operator((2, 3)).matrix, MO.identity_operator((2, 3)).matrix)
