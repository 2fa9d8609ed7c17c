"""GPU kernel parity against the CPU oracle (bit-exact for every kernel that
the reference computes deterministically)."""
import math

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_1504_06768_b200 import factor, liouville, ordering
from paper_1504_06768_b200 import _lib
from paper_1504_06768_b200.sparse import from_host, CSRMatrix
from tests.helpers import bits_equal, csr_equal, model, oracle_L

pytestmark = pytest.mark.gpu

SMALL = [("c1", {}), ("c4", {"i": 0}), ("c4", {"i": 300}), ("c2", {})]


def _host(o):
    return CSRMatrix(o.n, o.m, o.rp, o.ci, o.v)


@pytest.mark.parametrize("name,kw", SMALL)
def test_assembly_bit_exact(cuda, name, kw):
    H, c = model(name, **kw)
    L = liouville.build_liouvillian(H, c)
    assert csr_equal(L.matrix, oracle_L(H, c))


@pytest.mark.parametrize("name,kw", SMALL)
def test_shift_modify_bit_exact(cuda, name, kw):
    H, c = model(name, **kw)
    L = liouville.build_liouvillian(H, c)
    Lo = oracle_L(H, c)
    assert csr_equal(liouville.shift(L).matrix, O.shift(Lo))
    w = O.default_weight(Lo)
    mo, _, _ = O.build_modified(Lo, H.matrix.nrows, w)
    assert csr_equal(liouville.build_modified(L, w=w).matrix, mo)
    assert abs(liouville.default_weight(L) - w) <= 1e-12 * w


@pytest.mark.parametrize("name,kw", SMALL)
def test_rcm_bit_exact(cuda, name, kw):
    H, c = model(name, **kw)
    Lo = oracle_L(H, c)
    for m in (O.shift(Lo), O.build_modified(Lo, H.matrix.nrows)[0]):
        fwd, inv = O.rcm(m)
        p = ordering.rcm(from_host(_host(m)))
        assert bits_equal(p.forward, fwd) and bits_equal(p.inverse, inv)


@pytest.mark.parametrize("name,kw", SMALL)
def test_spmv_bit_exact(cuda, name, kw):
    H, c = model(name, **kw)
    Lo = oracle_L(H, c)
    x = np.random.default_rng(5).standard_normal(Lo.n) + 1j * np.random.default_rng(6).standard_normal(Lo.n)
    A = from_host(_host(Lo))
    y = torch.empty(Lo.n, dtype=torch.complex128, device="cuda")
    xd = torch.from_numpy(x).cuda()
    _lib.call("rs_csr_matvec", 1, A.n, _lib.ptr(A.row_ptr), _lib.ptr(A.col_idx),
              _lib.ptr(A.values), _lib.ptr(xd), _lib.ptr(y), _lib.stream_ptr())
    assert bits_equal(y.cpu().numpy(), O.csr_matvec(Lo, x))


def _rand_csr(rng, n, density, long_rows=(), empty_rows=()):
    """Random n x n CSR with sorted columns; some rows forced long / empty."""
    rows = []
    for r in range(n):
        if r in empty_rows:
            cols = np.empty(0, dtype=np.int64)
        elif r in long_rows:
            cols = np.arange(n, dtype=np.int64)
        else:
            cols = np.flatnonzero(rng.random(n) < density)
        rows.append(cols)
    rp = np.zeros(n + 1, dtype=np.int64)
    rp[1:] = np.cumsum([len(c) for c in rows])
    ci = np.concatenate(rows) if rp[-1] else np.empty(0, dtype=np.int64)
    v = rng.standard_normal(len(ci)) + 1j * rng.standard_normal(len(ci))
    return O.CSR(n, n, rp, ci, v)


@pytest.mark.parametrize("n,nsys,density,long_rows,empty_rows", [
    (7, 300, 0.4, (), (3,)),           # many systems inside one CTA
    (6000, 1, 0.0015, (17, 4000), (0, 5, 5999)),  # rows longer than a staging chunk
    (1600, 5, 0.005, (1599,), (0,)),   # CTAs straddling system boundaries
    (1, 3, 1.0, (), ()),
    # more 32-row groups than resident warps: each warp of the streamed
    # kernel walks several groups, groups straddle systems (n odd)
    (997, 100, 0.006, (500,), (0, 31, 32, 996)),
])
def test_spmv_random_batches_bit_exact(cuda, n, nsys, density, long_rows, empty_rows):
    rng = np.random.default_rng(n + nsys)
    mats = [_rand_csr(rng, n, density, long_rows, empty_rows) for _ in range(nsys)]
    A = from_host([_host(m) for m in mats])
    x = rng.standard_normal(n * nsys) + 1j * rng.standard_normal(n * nsys)
    y = torch.empty(n * nsys, dtype=torch.complex128, device="cuda")
    xd = torch.from_numpy(x).cuda()
    _lib.call("rs_csr_matvec", nsys, n, _lib.ptr(A.row_ptr), _lib.ptr(A.col_idx),
              _lib.ptr(A.values), _lib.ptr(xd), _lib.ptr(y), _lib.stream_ptr())
    ref = np.concatenate([O.csr_matvec(m, x[b * n:(b + 1) * n]) for b, m in enumerate(mats)])
    assert bits_equal(y.cpu().numpy(), ref)


@pytest.mark.parametrize("name,kw", SMALL)
def test_spmv_modified_bit_exact(cuda, name, kw):
    H, c = model(name, **kw)
    Lo = oracle_L(H, c)
    mo, _, _ = O.build_modified(Lo, H.matrix.nrows, O.default_weight(Lo))
    fwd, _ = O.rcm(mo)
    m = O.permute(mo, fwd)
    x = np.random.default_rng(9).standard_normal(m.n) + 1j * np.random.default_rng(10).standard_normal(m.n)
    A = from_host(_host(m))
    y = torch.empty(m.n, dtype=torch.complex128, device="cuda")
    _lib.call("rs_csr_matvec", 1, A.n, _lib.ptr(A.row_ptr), _lib.ptr(A.col_idx),
              _lib.ptr(A.values), _lib.ptr(torch.from_numpy(x).cuda()), _lib.ptr(y),
              _lib.stream_ptr())
    assert bits_equal(y.cpu().numpy(), O.csr_matvec(m, x))


FACTOR_CASES = [("c1", {}, 1e-5, 10.0), ("c1", {}, 0.0, math.inf), ("c1", {}, 1e-4, 300.0),
                ("c4", {"i": 0}, 0.0, math.inf), ("c2", {}, 1e-4, 300.0)]


@pytest.mark.parametrize("name,kw,d,p", FACTOR_CASES)
def test_factorize_bit_exact(cuda, name, kw, d, p):
    H, c = model(name, **kw)
    Lo = O.shift(oracle_L(H, c))
    fwd, _ = O.rcm(Lo)
    m = O.permute(Lo, fwd)
    fo = O.factorize_raw(m, d, p)
    f = factor.factor_batch(from_host(_host(m)), d, p)
    lp, li, lx, up, ui, ux, pinv = f.system_raw(0)
    assert bits_equal(lp, fo.Lp) and bits_equal(up, fo.Up) and bits_equal(pinv, fo.pinv)
    assert bits_equal(li, fo.Li) and bits_equal(ui, fo.Ui)
    assert bits_equal(lx, fo.Lx) and bits_equal(ux, fo.Ux)
    b = np.random.default_rng(9).standard_normal(m.n) + 0.5j
    assert bits_equal(factor.solve_lu(f, b), fo.solve(b))


def test_factorize_breakdown_step(cuda):
    """Reference breaks down at step n-1 on the shifted JC sweep (1e-5, 10)."""
    H, c = model("c4", i=0)
    Lo = O.shift(oracle_L(H, c))
    fwd, _ = O.rcm(Lo)
    m = O.permute(Lo, fwd)
    with pytest.raises(O.Breakdown) as e:
        O.factorize_raw(m, 1e-5, 10.0)
    with pytest.raises(factor.PreconditionerBreakdownError, match=f"step {e.value.step}$"):
        factor.ilutp(from_host(_host(m)), d=1e-5, p=10.0)


def test_factorize_overflow_resume(cuda):
    """Complete LU from a deliberately tiny capacity: the kernel stops at the
    first column that does not fit, the host grows the buffers and resumes;
    the result must still equal the reference factors bit for bit."""
    H, c = model("c2")
    Lo = O.shift(oracle_L(H, c))
    fwd, _ = O.rcm(Lo)
    m = O.permute(Lo, fwd)
    fo = O.factorize_raw(m, 0.0, math.inf)
    f = factor.factor_batch(from_host(_host(m)), 0.0, math.inf, capacity=m.n + 7)
    lp, li, lx, up, ui, ux, pinv = f.system_raw(0)
    assert bits_equal(lp, fo.Lp) and bits_equal(li, fo.Li) and bits_equal(lx, fo.Lx)
    assert bits_equal(up, fo.Up) and bits_equal(ui, fo.Ui) and bits_equal(ux, fo.Ux)


def test_factorize_batch_matches_single(cuda):
    """Block-diagonal batch (one CTA per system) == per-system reference."""
    mats = []
    for i in (0, 7, 300):
        H, c = model("c4", i=i)
        Lo = O.build_modified(oracle_L(H, c), 40)[0]
        fwd, _ = O.rcm(Lo)
        mats.append(O.permute(Lo, fwd))
    f = factor.factor_batch(from_host([_host(m) for m in mats]), 1e-5, 10.0)
    for b, m in enumerate(mats):
        fo = O.factorize_raw(m, 1e-5, 10.0)
        lp, li, lx, up, ui, ux, pinv = f.system_raw(b)
        assert bits_equal(lx, fo.Lx) and bits_equal(ux, fo.Ux) and bits_equal(li, fo.Li)
        x = np.random.default_rng(b).standard_normal(m.n) + 0j
        xs = np.zeros(3 * m.n, complex)
        xs[b * m.n:(b + 1) * m.n] = x
        got = factor.solve_lu(f, xs)[b * m.n:(b + 1) * m.n]
        assert bits_equal(got, fo.solve(x))


def test_rcm_random_corpus_bit_exact(cuda):
    """The 30 seeded random structures (some disconnected, isolated nodes) the
    reference ordered in tests/golden/make_golden.py, as one batch."""
    import os
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "rcm_corpus.npz"))
    k = 0
    while f"s{k}_n" in g:
        n = int(g[f"s{k}_n"])
        m = CSRMatrix(n, n, g[f"s{k}_rp"], g[f"s{k}_ci"], np.ones(len(g[f"s{k}_ci"])))
        p = ordering.rcm(from_host(m))
        assert bits_equal(p.inverse, g[f"s{k}_inv"]), k
        k += 1
    assert k == 30


@pytest.mark.parametrize("mixed", [False, True])
def test_rcm_batch_equals_single(cuda, mixed):
    """Shared-pattern batches (the c4 sweep) are ordered once; a batch mixing
    patterns (a trace-modified system) is ordered per system.  Both give
    every system the reference's permutation."""
    mats = [_host(O.shift(oracle_L(*model("c4", i=i)))) for i in (0, 100, 511)]
    if mixed:
        Lo = oracle_L(*model("c4", i=7))
        mo, _, _ = O.build_modified(Lo, 40, O.default_weight(Lo))
        mats.insert(1, _host(mo))
    A = from_host(mats)
    assert ordering.shared_structure(A) == (not mixed)
    fwd, inv = ordering.rcm_device(A)
    for b, m in enumerate(mats):
        f1, i1 = O.rcm(O.CSR(m.nrows, m.ncols, m.row_ptr, m.col_idx, m.values))
        sl = slice(b * m.nrows, (b + 1) * m.nrows)
        assert bits_equal(fwd[sl].cpu().numpy().astype(np.int64), f1)
        assert bits_equal(inv[sl].cpu().numpy().astype(np.int64), i1)


def test_vector_kernels(cuda):
    import ctypes
    n = 100_003
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(n, dtype=torch.complex128, device="cuda", generator=g)
    y = torch.randn(n, dtype=torch.complex128, device="cuda", generator=g)
    out = torch.empty(4, dtype=torch.float64, device="cuda")
    P = ctypes.c_void_p * 2
    _lib.call("rs_vdots", n, 2, P(x.data_ptr(), y.data_ptr()), P(y.data_ptr(), y.data_ptr()),
              _lib.ptr(out), _lib.stream_ptr())
    h = out.cpu().numpy()
    ref = np.vdot(x.cpu().numpy(), y.cpu().numpy())
    assert abs(complex(h[0], h[1]) - ref) <= 1e-12 * abs(ref) * 10
    assert abs(h[2] - np.vdot(y.cpu().numpy(), y.cpu().numpy()).real) <= 1e-10
    _lib.call("rs_amax", n, _lib.ptr(x), _lib.ptr(out), _lib.stream_ptr())
    assert out[0].item() == x.abs().max().item()
    z = torch.empty_like(x)
    c = (ctypes.c_double * 2)
    _lib.call("rs_lincomb", n, 2, P(x.data_ptr(), y.data_ptr()), c(2.0, 0.5), c(0.0, -1.0),
              _lib.ptr(z), _lib.stream_ptr())
    assert torch.allclose(z, 2 * x + (0.5 - 1j) * y, rtol=1e-14, atol=1e-14)


def test_block_extract(cuda):
    import ctypes
    H, c = model("c1")
    Lo = O.shift(oracle_L(H, c))
    A = from_host(_host(Lo))
    rp = torch.empty(401, dtype=torch.int32, device="cuda")
    nnz = ctypes.c_int64(0)
    _lib.call("rs_block_extract", 400, 100, 0, _lib.ptr(A.row_ptr), _lib.ptr(A.col_idx),
              _lib.ptr(A.values), _lib.ptr(rp), None, None, ctypes.byref(nnz), _lib.stream_ptr())
    ci = torch.empty(nnz.value, dtype=torch.int32, device="cuda")
    v = torch.empty(nnz.value, dtype=torch.complex128, device="cuda")
    _lib.call("rs_block_extract", 400, 100, 0, _lib.ptr(A.row_ptr), _lib.ptr(A.col_idx),
              _lib.ptr(A.values), _lib.ptr(rp), _lib.ptr(ci), _lib.ptr(v), ctypes.byref(nnz),
              _lib.stream_ptr())
    d = Lo.dense()
    got = np.zeros((400, 400), complex)
    rph = rp.cpu().numpy()
    for r in range(400):
        b = r // 100
        for q in range(rph[r], rph[r + 1]):
            got[r, b * 100 + ci[q].item()] = v[q].item()
    want = np.zeros_like(d)
    for b in range(4):
        want[b * 100:(b + 1) * 100, b * 100:(b + 1) * 100] = d[b * 100:(b + 1) * 100,
                                                                b * 100:(b + 1) * 100]
    assert bits_equal(got, want)


def _solve_both_paths(f, b):
    """M^{-1} b through the column-stream sweeps and the row-oriented sweeps."""
    assert f.csc
    xc = factor.solve_lu(f, b)
    f.csc = False
    try:
        xr = factor.solve_lu(f, b)
    finally:
        f.csc = True
    return xc, xr


@pytest.mark.parametrize("name,kw,d,p", [("c2", {}, 0.0, math.inf), ("c2", {}, 1e-4, 300.0),
                                         ("c1", {}, 1e-5, 10.0), ("c4", {"i": 9}, 0.0, math.inf)])
def test_apply_column_stream_bit_exact(cuda, name, kw, d, p):
    """The column-stream apply (colsweep.cuh: columns > 64 entries span several
    stream rows; c2 complete LU streams far more rows than the shared ring
    holds) equals the reference lower/upper column loops bit for bit, and so
    does the row-oriented sweep."""
    H, c = model(name, **kw)
    Lo = O.shift(oracle_L(H, c))
    fwd, _ = O.rcm(Lo)
    m = O.permute(Lo, fwd)
    fo = O.factorize_raw(m, d, p)
    f = factor.factor_batch(from_host(_host(m)), d, p)
    b = np.random.default_rng(11).standard_normal(m.n) - 0.25j
    ref = fo.solve(b)
    xc, xr = _solve_both_paths(f, b)
    assert bits_equal(xc, ref) and bits_equal(xr, ref)


def test_apply_column_stream_random_long_columns(cuda):
    """Random unsymmetric sparse matrix with a few dense columns (a single
    column longer than the whole staging ring) and empty L / U columns."""
    rng = np.random.default_rng(3)
    n = 3000
    mats = []
    for dense_cols in ((5, 2100), (0, 2999)):
        M = _rand_csr(rng, n, 0.002, long_rows=(), empty_rows=())
        rows = [list(M.ci[M.rp[r]:M.rp[r + 1]]) for r in range(n)]
        for r in range(n):
            rows[r] = sorted(set(rows[r]) | {r} | ({dc for dc in dense_cols if r % 3 == 0}))
        rp = np.zeros(n + 1, dtype=np.int64)
        rp[1:] = np.cumsum([len(x) for x in rows])
        ci = np.concatenate([np.asarray(x, dtype=np.int64) for x in rows])
        v = rng.standard_normal(len(ci)) + 1j * rng.standard_normal(len(ci))
        v[rp[:-1] + np.array([rows[r].index(r) for r in range(n)])] += 40.0  # diagonal dominance
        mats.append(O.CSR(n, n, rp, ci, v))
    f = factor.factor_batch(from_host([_host(m) for m in mats]), 0.0, math.inf)
    b = rng.standard_normal(2 * n) + 1j * rng.standard_normal(2 * n)
    xc, xr = _solve_both_paths(f, b)
    for k, m in enumerate(mats):
        ref = O.factorize_raw(m, 0.0, math.inf).solve(b[k * n:(k + 1) * n])
        assert bits_equal(xc[k * n:(k + 1) * n], ref)
        assert bits_equal(xr[k * n:(k + 1) * n], ref)


@pytest.mark.parametrize("name,kw,d,p,cps,nsys", [("c2", {}, 1e-4, 300.0, 4, 1),
                                                  ("c2", {}, 0.0, math.inf, 3, 1),
                                                  ("c4", {"i": 77}, 0.0, math.inf, 2, 3)])
def test_factorize_multi_cta_bit_exact(cuda, monkeypatch, name, kw, d, p, cps, nsys):
    """Multi-CTA factorization (one system across several co-resident CTAs,
    used by default for n >= 8192) forced onto systems the oracle factors in
    seconds: factors and the apply equal the reference bit for bit."""
    monkeypatch.setenv("RHOSOLVE_ILU_CPS", str(cps))
    H, c = model(name, **kw)
    Lo = O.shift(oracle_L(H, c))
    fwd, _ = O.rcm(Lo)
    m = O.permute(Lo, fwd)
    fo = O.factorize_raw(m, d, p)
    f = factor.factor_batch(from_host([_host(m)] * nsys), d, p)
    b = np.random.default_rng(4).standard_normal(m.n * nsys) + 0.1j
    x = factor.solve_lu(f, b)
    for s in range(nsys):
        lp, li, lx, up, ui, ux, pinv = f.system_raw(s)
        assert bits_equal(lp, fo.Lp) and bits_equal(up, fo.Up) and bits_equal(pinv, fo.pinv)
        assert bits_equal(li, fo.Li) and bits_equal(ui, fo.Ui)
        assert bits_equal(lx, fo.Lx) and bits_equal(ux, fo.Ux)
        assert bits_equal(x[s * m.n:(s + 1) * m.n], fo.solve(b[s * m.n:(s + 1) * m.n]))


def test_apply_sliding_window_multi_consumer_bit_exact(cuda, monkeypatch):
    """A lone system whose sweep vector does not fit shared memory (n = 14,400)
    sweeps through the sliding shared-memory window with several consumer
    warps (colsweep.cuh col_consume_win): same bits as the oracle's column
    loops, with the window on or off and for 1, 3 and 6 consumers."""
    from paper_1504_06768_b200 import configs
    monkeypatch.setenv("RHOSOLVE_GRID_MIN_N", "100000000")
    H, c = configs.optomech(n_c=4, n_m=30)
    Lo = oracle_L(H, c)
    S = O.shift(Lo)
    fwd, _ = O.rcm(S)
    pm = O.permute(S, fwd)
    assert pm.n == 14400
    fo = O.factorize_raw(pm, 1e-3, 8.0)
    f = factor.factor_batch(from_host(_host(pm)), 1e-3, 8.0)
    rng = np.random.default_rng(3)
    b = rng.standard_normal(pm.n) + 1j * rng.standard_normal(pm.n)
    ref = fo.solve(b)
    f.ensure_cols()
    assert 0 < f.reach < pm.n
    for win in ("1", "0"):
        monkeypatch.setenv("RHOSOLVE_COL_WINDOW", win)
        for w in ("1", "3", "6"):
            monkeypatch.setenv("RHOSOLVE_COL_CONSUMERS", w)
            assert bits_equal(factor.solve_lu(f, b), ref), (win, w)


def test_shared_structure_detection(cuda):
    """ordering.shared_structure: one RCM for a batch whose systems store
    system 0's pattern; any differing row extent or column index disables it
    (rs_same_pattern: one kernel, one flag)."""
    import torch
    from paper_1504_06768_b200 import ordering
    from paper_1504_06768_b200.sparse import DeviceCSR
    rp1 = torch.tensor([0, 2, 3, 5], dtype=torch.int32, device="cuda")
    ci1 = torch.tensor([0, 2, 1, 0, 2], dtype=torch.int32, device="cuda")

    def batch(rps, cis):
        rp, ci, base = [], [], 0
        for r, c in zip(rps, cis):
            rp.append(r[:-1] + base)
            ci.append(c)
            base += int(r[-1])
        rp.append(torch.tensor([base], dtype=torch.int32, device="cuda"))
        ci = torch.cat(ci)
        return DeviceCSR(3, len(rps), torch.cat(rp), ci,
                         torch.zeros(ci.numel(), dtype=torch.complex128, device="cuda"))

    assert ordering.shared_structure(batch([rp1] * 3, [ci1] * 3))
    assert not ordering.shared_structure(batch([rp1], [ci1]))  # a single system
    ci2 = torch.tensor([0, 2, 1, 1, 2], dtype=torch.int32, device="cuda")      # same extents, other column
    assert not ordering.shared_structure(batch([rp1, rp1], [ci1, ci2]))
    rp3 = torch.tensor([0, 1, 3, 5], dtype=torch.int32, device="cuda")         # same nnz, other extents
    ci3 = torch.tensor([0, 1, 2, 0, 2], dtype=torch.int32, device="cuda")
    assert not ordering.shared_structure(batch([rp1, rp3], [ci1, ci3]))
    rp4 = torch.tensor([0, 1, 2, 3], dtype=torch.int32, device="cuda")         # other nnz
    ci4 = torch.tensor([0, 1, 2], dtype=torch.int32, device="cuda")
    assert not ordering.shared_structure(batch([rp1, rp4], [ci1, ci4]))
