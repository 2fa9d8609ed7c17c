"""End-to-end steady-state parity on the GPU against the oracle (reference
algorithm on CPU): trace distance <= 1e-6 and ||L vec rho||_2 <= 1e-10."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1504_06768_b200 import liouville, steady
from tests.helpers import bits_equal, model, oracle_L

pytestmark = pytest.mark.gpu


def _check(res, ref, resid=1e-10):
    assert res.residual <= resid
    assert O.trace_distance(res.rho, ref["rho"]) <= 1e-6


def test_c1_inverse_power_direct(cuda):
    H, c = model("c1")
    L = liouville.build_liouvillian(H, c)
    ref = O.inverse_power(oracle_L(H, c), 20, tol=1e-12, inner="direct", seed=0)
    res = steady.inverse_power(L, tol=1e-12, inner="direct", ordering_name="rcm", seed=0)
    _check(res, ref)
    assert res.iterations == ref["outer"]


def test_c1_inverse_power_bicgstab(cuda):
    H, c = model("c1")
    L = liouville.build_liouvillian(H, c)
    ref = O.inverse_power(oracle_L(H, c), 20, tol=1e-12, inner="iterative", solver="bicgstab",
                          d=1e-5, p=10, seed=0)
    res = steady.inverse_power(L, tol=1e-12, inner="iterative", ordering_name="rcm",
                               solver="bicgstab", d=1e-5, p=10, seed=0)
    _check(res, ref)


def test_c1_inverse_power_gmres(cuda):
    H, c = model("c1")
    L = liouville.build_liouvillian(H, c)
    ref = O.inverse_power(oracle_L(H, c), 20, tol=1e-12, inner="iterative", solver="gmres",
                          d=1e-5, p=10, seed=0)
    res = steady.inverse_power(L, tol=1e-12, inner="iterative", ordering_name="rcm",
                               solver="gmres", d=1e-5, p=10, seed=0)
    _check(res, ref)


@pytest.mark.parametrize("method", ["bicgstab", "gmres", "direct"])
def test_c1_linear(cuda, method):
    H, c = model("c1")
    L = liouville.build_liouvillian(H, c)
    ref = O.solve_linear(oracle_L(H, c), 20, method=method, d=1e-5, p=10, tol=1e-12)
    if method == "direct":
        res = steady.solve_direct(L, "rcm")
    else:
        res = steady.solve_iterative(L, "rcm", method, d=1e-5, p=10, tol=1e-12)
        assert res.converged == ref["converged"]
    _check(res, ref)


def test_c2_inverse_power_bicgstab_defaults(cuda):
    H, c = model("c2")
    L = liouville.build_liouvillian(H, c)
    ref = O.inverse_power(oracle_L(H, c), 80, tol=1e-12, inner="iterative", solver="bicgstab",
                          d=1e-4, p=300, seed=1)
    res = steady.inverse_power(L, tol=1e-12, inner="iterative", ordering_name="rcm",
                               solver="bicgstab", d=1e-4, p=300, seed=1)
    _check(res, ref)


def test_c4_batch_power_direct(cuda):
    idx = [0, 100, 255, 511]
    models = [model("c4", i=i) for i in idx]
    L = liouville.build_liouvillian_batch(models)
    res = steady.inverse_power_batch(L, [2 + i for i in idx], tol=1e-12, inner="direct",
                                     ordering_name="rcm")
    for (H, c), i, r in zip(models, idx, res):
        ref = O.inverse_power(oracle_L(H, c), 40, tol=1e-12, inner="direct", seed=2 + i)
        assert r.error is None
        _check(r, ref)


@pytest.mark.parametrize("ordering_name", ["rcm", "natural"])
def test_c4_batch_from_pinned_host_buffers(cuda, ordering_name):
    """The end-to-end path of bench.py: a PinnedBatchCSR (host) input, values
    uploaded on the side stream while the pattern is RCM-ordered, gives the
    same bits as the device-resident input."""
    from paper_1504_06768_b200.sparse import pin_batch
    idx = [0, 7, 300, 511]
    L = liouville.build_liouvillian_batch([model("c4", i=i) for i in idx])
    seeds = [2 + i for i in idx]
    kw = dict(tol=1e-12, inner="direct", ordering_name=ordering_name)
    dev = steady.inverse_power_batch(L, seeds, **kw)
    pinned = pin_batch([L.matrix.system(b) for b in range(L.nsys)])
    host = steady.inverse_power_batch(liouville.LiouvillianSystem(pinned, 40, "plain"), seeds, **kw)
    for a, b in zip(dev, host):
        assert a.error is None and b.error is None
        assert bits_equal(a.rho, b.rho)
        assert a.residual == b.residual


@pytest.mark.slow
def test_c3_inverse_power_bicgstab_defaults(cuda):
    """Optomechanics 6x40 (n = 57,600): inverse power with ILUTP(1e-4, 300)
    BiCGStab under RCM, against the rho the reference itself produced."""
    import os
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "c3.npz"))
    H, c = model("c3")
    L = liouville.build_liouvillian(H, c)
    res = steady.inverse_power(L, tol=1e-12, inner="iterative", ordering_name="rcm",
                               solver="bicgstab", d=1e-4, p=300.0)
    assert res.residual <= 1e-10
    assert O.trace_distance(res.rho, g["power_bicgstab_rho"]) <= 1e-6


def test_sharded_path_single_gpu_kerr_kerr(cuda):
    """Config-5 code path (row-sharded driver, block-Jacobi ILUTP, grid-wide
    BiCGStab) at N=8 on one GPU, against the oracle's direct inverse power."""
    from paper_1504_06768_b200 import configs, sharded
    H, c = configs.kerr_kerr(N=8)
    L = liouville.build_liouvillian(H, c)
    res = sharded.inverse_power_sharded(L, tol=1e-10, d=1e-5, p=10.0, seed=3, blocks=2)
    ref = O.inverse_power(oracle_L(H, c), 64, tol=1e-12, inner="direct", seed=3)
    assert res.residual <= 1e-10
    assert O.trace_distance(res.rho, ref["rho"]) <= 1e-6


def test_c3_solve_direct(cuda):
    """complete LU of the trace-modified optomechanics
    Liouvillian (n = 57,600, fill ~184; multi-CTA factorization) -- the
    reference needs 200-250 s for it."""
    import os
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "c3.npz"))
    H, c = model("c3")
    L = liouville.build_liouvillian(H, c)
    res = steady.solve_direct(L, ordering_name="rcm")
    assert res.residual <= 1e-10
    assert O.trace_distance(res.rho, g["power_bicgstab_rho"]) <= 1e-6


def test_c4_two_shards_equal_one_batch(cuda):
    """The N-GPU sweep is the 1-GPU sweep cut into contiguous shards: solving
    two shards separately gives, system by system, the bits of the one batch."""
    idx = list(range(248, 264))
    models = [model("c4", i=i) for i in idx]
    kw = dict(tol=1e-12, inner="direct", ordering_name="rcm")
    whole = steady.inverse_power_batch(liouville.build_liouvillian_batch(models),
                                       [2 + i for i in idx], **kw)
    halves = []
    for lo in (0, 8):
        L = liouville.build_liouvillian_batch(models[lo:lo + 8])
        halves += steady.inverse_power_batch(L, [2 + i for i in idx[lo:lo + 8]], **kw)
    for a, b in zip(whole, halves):
        assert a.error is None and b.error is None
        assert bits_equal(a.rho, b.rho) and a.iterations == b.iterations
