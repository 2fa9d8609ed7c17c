"""Compact complete-LU kernel (csrc/ilu_compact.cu: the working column of every
warp by position in shared memory) against the reference factorize
(_ckernels.pyx:144-385, d = 0, no cap) through the oracle, bit for bit, and
against the general column pipeline (csrc/ilu.cu) on larger batches: every
planner branch (16 / 8 / 7 warps per system, byte and int32 row maps), the
fall-back when a column outgrows the shared-memory capacity, pivot ties,
stored zeros and zero pivots."""
import math

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_1504_06768_b200 import _lib, configs, factor, liouville, ordering
from paper_1504_06768_b200.sparse import from_host
from tests.helpers import bits_equal
from tests.test_gpu_frontal import _c4, _check, _host, _random_system

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _compact_on(monkeypatch):
    monkeypatch.delenv("RHOSOLVE_FRONTAL", raising=False)
    monkeypatch.setenv("RHOSOLVE_COMPACT", "1")


def _compact_taken():
    return int(_lib.load().rs_debug_compact_taken())


def _c4_batch_device(count):
    L = liouville.build_liouvillian_batch([configs.jc_sweep(i) for i in range(count)])
    sh = liouville.shift(L)
    fwd, inv = ordering.rcm_device(sh.matrix)
    return ordering.permute(sh.matrix, fwd, inv)


def _same_factors(a, b):
    n, B = a.n, a.nsys
    assert torch.equal(a.pinv, b.pinv)
    assert torch.equal(a.raw[0], b.raw[0]) and torch.equal(a.raw[3], b.raw[3])  # Lp, Up
    lp = a.raw[0].view(B, n + 1).cpu()
    up = a.raw[3].view(B, n + 1).cpu()
    for s in range(B):
        for (ia, xa, ib, xb, cnt) in ((a.raw[1], a.raw[2], b.raw[1], b.raw[2], int(lp[s, n])),
                                      (a.raw[4], a.raw[5], b.raw[4], b.raw[5], int(up[s, n]))):
            lo = s * (ia.numel() // B)
            lob = s * (ib.numel() // B)
            assert torch.equal(ia[lo:lo + cnt], ib[lob:lob + cnt]), s
            assert torch.equal(torch.view_as_real(xa[lo:lo + cnt]).view(torch.int64),
                               torch.view_as_real(xb[lob:lob + cnt]).view(torch.int64)), s


def test_compact_c4_batch_bit_exact(cuda):
    idx = [0, 1, 100, 255, 256, 300, 511]
    mats = [_c4(i) for i in idx]
    f = factor.factor_batch(from_host([_host(m) for m in mats]), 0.0, math.inf)
    assert _compact_taken() == 1
    for b, m in enumerate(mats):
        _check(f, b, m)


def test_compact_modified_and_small_systems(cuda):
    from tests.helpers import model, oracle_L
    H, c = model("c1")
    Lo = O.shift(oracle_L(H, c))
    fwd, _ = O.rcm(Lo)
    for m in (O.permute(Lo, fwd), _c4(17, modified=True)):
        f = factor.factor_batch(from_host(_host(m)), 0.0, math.inf)
        assert _compact_taken() == 1
        _check(f, 0, m)


@pytest.mark.parametrize("count", [160, 300, 512])
def test_compact_equals_general_pipeline(cuda, monkeypatch, count):
    """16 warps x 2 per SM (160), 8 warps x 3 per SM (300), 7 warps x 4 per SM (512)."""
    A = _c4_batch_device(count)
    a = factor.factor_batch(A, 0.0, math.inf)
    assert _compact_taken() == 1
    monkeypatch.setenv("RHOSOLVE_COMPACT", "0")
    monkeypatch.setenv("RHOSOLVE_FRONTAL", "0")
    b = factor.factor_batch(A, 0.0, math.inf)
    assert _compact_taken() == 0
    _same_factors(a, b)


@pytest.mark.parametrize("knob", [("RHOSOLVE_COMPACT_NOPOS8", "1"), ("RHOSOLVE_COMPACT_CAPX", "64"),
                                  ("RHOSOLVE_COMPACT_CAPX", "160")])
def test_compact_variants_and_capacity_fallback(cuda, monkeypatch, knob):
    """int32 row map in global scratch; a shared-memory capacity below the
    columns' patterns (64: every system, 160: late columns) hands the system
    to the general kernel -- same factors either way."""
    idx = [3, 200, 410]
    mats = [_c4(i) for i in idx]
    monkeypatch.setenv(*knob)
    f = factor.factor_batch(from_host([_host(m) for m in mats]), 0.0, math.inf)
    assert _compact_taken() == 1
    for b, m in enumerate(mats):
        _check(f, b, m)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_compact_random_batch(cuda, seed):
    rng = np.random.default_rng(seed)
    n = 120
    mats = [_random_system(rng, n, band=int(rng.integers(3, 20)), density=rng.uniform(0.1, 0.6),
                           ints=bool(k % 2)) for k in range(12)]
    f = factor.factor_batch(from_host([_host(m) for m in mats]), 0.0, math.inf,
                            raise_on_fail=False)
    assert _compact_taken() == 1
    for b, m in enumerate(mats):
        try:
            O.factorize_raw(m, 0.0, math.inf)
        except O.Breakdown as e:
            assert f.fail[b] == e.step
            continue
        assert f.fail[b] < 0
        _check(f, b, m)


def test_compact_zero_pivot_in_batch(cuda):
    good = _c4(5)
    n = good.n
    v = good.v.copy()
    v[good.ci == 5] = 0.0
    bad = O.CSR(n, n, good.rp, good.ci, v)
    with pytest.raises(O.Breakdown) as e:
        O.factorize_raw(bad, 0.0, math.inf)
    f = factor.factor_batch(from_host([_host(good), _host(bad), _host(good)]), 0.0, math.inf,
                            raise_on_fail=False)
    assert _compact_taken() == 1
    assert list(f.fail) == [-1, e.value.step, -1]
    _check(f, 0, good)
    _check(f, 2, good)


def test_compact_output_overflow_resumes(cuda):
    """Complete LU whose first output capacity is too small: the compact kernel
    reports the overflow column and the grown buffers are finished by the
    general kernel's resume -- the reference's factors in the end."""
    m = _c4(40)
    f = factor.factor_batch(from_host(_host(m)), 0.0, math.inf, capacity=20000)
    _check(f, 0, m)


def test_hybrid_frontal_pipeline_split_same_factors(cuda, monkeypatch):
    """The measured-and-disabled experiment of DESIGN.md (RHOSOLVE_HYBRID_F: the
    first F systems in the 64-register frontal build, the rest in pipeline CTAs
    without shared-memory state on a side stream) still produces the factors
    of the default path."""
    A = _c4_batch_device(12)
    a = factor.factor_batch(A, 0.0, math.inf)
    monkeypatch.setenv("RHOSOLVE_HYBRID_F", "5")
    b = factor.factor_batch(A, 0.0, math.inf)
    assert _compact_taken() == 0 and int(_lib.load().rs_debug_frontal_taken()) == 5
    _same_factors(a, b)


@pytest.mark.parametrize("n", [1, 2, 5, 33, 64])
def test_compact_tiny_systems(cuda, n):
    """Orders around and below a warp: n = 1 (a lone pivot), a full 2 x 2, ragged
    bands -- the planner's capacities clamp to n and the factors stay the oracle's."""
    rng = np.random.default_rng(100 + n)
    mats = [_random_system(rng, n, band=max(1, min(n - 1, int(rng.integers(1, 6)))), density=0.7,
                           ints=bool(k % 2)) for k in range(6)]
    f = factor.factor_batch(from_host([_host(m) for m in mats]), 0.0, math.inf,
                            raise_on_fail=False)
    assert _compact_taken() == 1
    for b, m in enumerate(mats):
        try:
            O.factorize_raw(m, 0.0, math.inf)
        except O.Breakdown as e:
            assert f.fail[b] == e.step
            continue
        assert f.fail[b] < 0
        _check(f, b, m)
