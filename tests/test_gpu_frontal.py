"""Right-looking frontal complete LU (csrc/frontal.cu) against the reference
factorize (_ckernels.pyx:144-385, d = 0, no cap) through the oracle, bit for
bit: Lp/Li/Lx/Up/Ui/Ux/pinv of every system, including pivot ties, explicit
zeros, per-system structures in one batch and zero pivots (handed to the
column pipeline, which must report the reference's step)."""
import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_1504_06768_b200 import _lib, factor
from paper_1504_06768_b200.sparse import CSRMatrix, from_host
from tests.helpers import bits_equal, model, oracle_L

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _frontal_on(monkeypatch):
    # the frontal kernel is opt-in (csrc/frontal.cu: frontal_enabled)
    monkeypatch.setenv("RHOSOLVE_FRONTAL", "1")


def _host(o):
    return CSRMatrix(o.n, o.m, o.rp, o.ci, o.v)


def _taken():
    return int(_lib.load().rs_debug_frontal_taken())


def _check(f, b, m):
    fo = O.factorize_raw(m, 0.0, math.inf)
    lp, li, lx, up, ui, ux, pinv = f.system_raw(b)
    assert bits_equal(lp, fo.Lp) and bits_equal(up, fo.Up), b
    assert bits_equal(pinv, fo.pinv), b
    assert bits_equal(li, fo.Li) and bits_equal(ui, fo.Ui), b
    assert bits_equal(lx, fo.Lx) and bits_equal(ux, fo.Ux), b


def _c4(i, modified=False):
    H, c = model("c4", i=i)
    L = oracle_L(H, c)
    Lo = O.build_modified(L, 40)[0] if modified else O.shift(L)
    fwd, _ = O.rcm(Lo)
    return O.permute(Lo, fwd)


def test_frontal_c4_batch_bit_exact(cuda):
    idx = [0, 1, 100, 255, 256, 300, 511]
    mats = [_c4(i) for i in idx]
    f = factor.factor_batch(from_host([_host(m) for m in mats]), 0.0, math.inf)
    assert _taken() == len(mats)
    for b, m in enumerate(mats):
        _check(f, b, m)


@pytest.mark.parametrize("name", ["c1", "c4m"])
def test_frontal_other_systems(cuda, name):
    if name == "c1":
        H, c = model("c1")
        Lo = O.shift(oracle_L(H, c))
        fwd, _ = O.rcm(Lo)
        m = O.permute(Lo, fwd)
    else:
        m = _c4(17, modified=True)
    f = factor.factor_batch(from_host(_host(m)), 0.0, math.inf)
    _check(f, 0, m)


def test_frontal_matches_pipeline(cuda, monkeypatch):
    mats = [_c4(i) for i in range(0, 512, 37)]
    dm = from_host([_host(m) for m in mats])
    a = factor.factor_batch(dm, 0.0, math.inf)
    assert _taken() == len(mats)
    monkeypatch.setenv("RHOSOLVE_FRONTAL", "0")
    bb = factor.factor_batch(dm, 0.0, math.inf)
    assert _taken() == 0
    for s in range(len(mats)):
        for x, y in zip(a.system_raw(s), bb.system_raw(s)):
            assert bits_equal(x, y)


def _random_system(rng, n, band, density, ints):
    """Random banded structure with a full diagonal; integer-valued entries
    make pivot magnitudes tie (the lowest original row must win)."""
    r, c = [], []
    for i in range(n):
        lo, hi = max(0, i - band), min(n, i + band + 1)
        cols = [j for j in range(lo, hi) if j == i or rng.random() < density]
        r += [i] * len(cols)
        c += cols
    r, c = np.array(r), np.array(c)
    if ints:
        v = rng.integers(-2, 3, len(r)) + 1j * rng.integers(-1, 2, len(r))
        v[r == c] = np.where(v[r == c] == 0, 1.0, v[r == c])
        v = v.astype(complex)
    else:
        v = rng.standard_normal(len(r)) + 1j * rng.standard_normal(len(r))
    # a few explicit zeros stay stored (structure, not value, drives fill)
    z = rng.random(len(r)) < 0.03
    v[z & (r != c)] = 0.0
    return O.coo_to_csr(n, n, r, c, v, prune=False)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_frontal_random_batch(cuda, seed):
    rng = np.random.default_rng(seed)
    n = 120
    mats = [_random_system(rng, n, band=int(rng.integers(3, 20)), density=rng.uniform(0.1, 0.6),
                           ints=bool(k % 2)) for k in range(12)]
    f = factor.factor_batch(from_host([_host(m) for m in mats]), 0.0, math.inf,
                            raise_on_fail=False)
    assert _taken() >= 1
    for b, m in enumerate(mats):
        try:
            O.factorize_raw(m, 0.0, math.inf)
        except O.Breakdown as e:
            assert f.fail[b] == e.step
            continue
        assert f.fail[b] < 0
        _check(f, b, m)


def test_frontal_zero_pivot_in_batch(cuda):
    """A numerically singular system among regular ones: the frontal kernel
    leaves it to the column pipeline, which reports the reference's step."""
    good = _c4(5)
    n = good.n
    # column 5 keeps its structure but holds only stored zeros: every update
    # into it is a product with 0, so its pivot is exactly zero
    v = good.v.copy()
    v[good.ci == 5] = 0.0
    bad = O.CSR(n, n, good.rp, good.ci, v)
    with pytest.raises(O.Breakdown) as e:
        O.factorize_raw(bad, 0.0, math.inf)
    f = factor.factor_batch(from_host([_host(good), _host(bad), _host(good)]), 0.0, math.inf,
                            raise_on_fail=False)
    assert list(f.fail) == [-1, e.value.step, -1]
    _check(f, 0, good)
    _check(f, 2, good)
