"""Round-2 parity cases on fixtures the reference itself produced
(tests/golden/*.npz): condest, the config-2 plain iterative solve, config-3
RCM and GMRES(20) inverse power, permute, natural-order direct solve, the
'cmd' ordering away from sigma ~ 0, column-pre-ordered Krylov
preconditioners, trace output, and per-system failures in a batch."""
import io
import os

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_1504_06768_b200 import _lib, configs, factor, krylov, liouville, ordering, steady
from paper_1504_06768_b200.sparse import CSRMatrix, DeviceCSR, Permutation, from_host
from tests.helpers import bits_equal, csr_equal, model, oracle_L

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def G(name):
    return np.load(os.path.join(GOLD, f"{name}.npz"))


def _host(o):
    return CSRMatrix(o.n, o.m, o.rp, o.ci, o.v)


def _rel(a, b):
    return abs(a - b) / abs(b)


# ---- a9 condest (factor.py:152-157) -----------------------------------------
@pytest.mark.parametrize("key,variant,d,p", [
    ("f_sh_1e5_10", "shift", 1e-5, 10.0), ("f_sh_lu", "shift", 0.0, float("inf")),
    ("f_mod_1e5_10", "mod", 1e-5, 10.0)])
def test_c1_condest_matches_reference(cuda, key, variant, d, p):
    g = G("c1")
    H, c = model("c1")
    Lo = oracle_L(H, c)
    m = O.shift(Lo) if variant == "shift" else O.build_modified(Lo, 20, float(g["w"]))[0]
    fwd = g["rcm_shift_fwd"] if variant == "shift" else g["rcm_mod_fwd"]
    A = from_host(_host(O.permute(m, fwd)))
    f = factor.lu(A) if d == 0.0 else factor.ilutp(A, d, p)
    # the apply is bit-exact; |.| is hypot on both sides
    assert _rel(factor.condest(f), float(g[key + "_condest"])) <= 1e-13


def test_c1_c2_solver_condest_matches_reference(cuda):
    g1, g2 = G("c1"), G("c2")
    H, c = model("c1")
    L = liouville.build_liouvillian(H, c)
    r = steady.solve_iterative(L, "rcm", "bicgstab", d=1e-5, p=10, tol=1e-12)
    assert _rel(r.condest, float(g1["bicgstab_condest"])) <= 1e-12
    assert r.iterations == int(g1["bicgstab_iterations"])
    r = steady.solve_iterative(L, "rcm", "gmres", d=1e-5, p=10, tol=1e-12)
    assert _rel(r.condest, float(g1["gmres_condest"])) <= 1e-12
    assert r.iterations == int(g1["gmres_iterations"])
    r = steady.inverse_power(L, tol=1e-12, inner="iterative", ordering_name="rcm",
                             solver="bicgstab", d=1e-5, p=10, seed=0)
    assert _rel(r.condest, float(g1["power_bicgstab_condest"])) <= 1e-12
    assert r.iterations == int(g1["power_bicgstab_iterations"])
    H, c = model("c2")
    L = liouville.build_liouvillian(H, c)
    r = steady.inverse_power(L, tol=1e-12, inner="iterative", ordering_name="rcm",
                             solver="bicgstab", d=1e-4, p=300.0, seed=1)
    assert _rel(r.condest, float(g2["power_bicgstab_condest"])) <= 1e-10
    assert r.iterations == int(g2["power_bicgstab_iterations"])
    assert O.trace_distance(r.rho, g2["power_bicgstab_rho"]) <= 1e-6


# ---- a17: config 2's plain iterative solve (BASELINE config 2) ---------------
def test_c2_solve_iterative_1e5_10(cuda):
    g = G("c2")
    H, c = model("c2")
    L = liouville.build_liouvillian(H, c)
    r = steady.solve_iterative(L, "rcm", "bicgstab", d=1e-5, p=10, tol=1e-12)
    ref = O.solve_linear(oracle_L(H, c), 80, method="bicgstab", d=1e-5, p=10, tol=1e-12)
    assert r.iterations == int(g["bicgstab_1e5_10_iterations"])
    assert r.converged == ref["converged"] and not r.breakdown
    assert r.residual <= 1e-10
    assert O.trace_distance(r.rho, g["bicgstab_1e5_10_rho"]) <= 1e-6
    assert _rel(r.fill_factor, float(g["bicgstab_1e5_10_fill"])) <= 1e-14
    assert _rel(r.condest, float(g["bicgstab_1e5_10_condest"])) <= 1e-10


def test_c2_shifted_ilutp_breakdown_step(cuda):
    """ILUTP(1e-5, 10) of config 2's RCM-ordered shifted matrix breaks down at
    the step the reference reports."""
    g = G("c2")
    H, c = model("c2")
    L = liouville.build_liouvillian(H, c)
    with pytest.raises(factor.PreconditionerBreakdownError) as e:
        steady.inverse_power(L, tol=1e-12, inner="iterative", ordering_name="rcm",
                             solver="bicgstab", d=1e-5, p=10.0, seed=1)
    assert str(e.value) == f"zero pivot at elimination step {int(g['f_sh_1e5_10_fail'])}"


# ---- a4: RCM of config 3 (the weak-RCM configuration), bit-exact -------------
def test_c3_rcm_bit_exact_vs_reference(cuda):
    g = G("c3")
    H, c = model("c3")
    L = liouville.build_liouvillian(H, c)
    p = ordering.rcm(liouville.shift(L).matrix)
    assert bits_equal(p.forward, g["rcm_shift_fwd"]) and bits_equal(p.inverse, g["rcm_shift_inv"])
    p = ordering.rcm(liouville.build_modified(L, w=float(g["w"])).matrix)
    assert bits_equal(p.forward, g["rcm_mod_fwd"]) and bits_equal(p.inverse, g["rcm_mod_inv"])
    # the default weight the reference derived (numpy pairwise mean) to 1e-12
    assert _rel(liouville.default_weight(L), float(g["w"])) <= 1e-12


# ---- a5: sparse.permute (sparse.py:276-282), bit-exact -----------------------
@pytest.mark.parametrize("name,kw", [("c1", {}), ("c4", {"i": 300}), ("c2", {})])
def test_permute_bit_exact(cuda, name, kw):
    H, c = model(name, **kw)
    Lo = oracle_L(H, c)
    for m in (O.shift(Lo), O.build_modified(Lo, H.matrix.nrows)[0]):
        fwd, inv = O.rcm(m)
        A = from_host(_host(m))
        f32 = torch.from_numpy(fwd.astype(np.int32)).cuda()
        i32 = torch.from_numpy(inv.astype(np.int32)).cuda()
        assert csr_equal(ordering.permute(A, f32, i32), O.permute(m, fwd))
    # an arbitrary (non-RCM) permutation of a batch of two systems
    rng = np.random.default_rng(4)
    m = O.shift(Lo)
    perms = [rng.permutation(m.n) for _ in range(2)]
    A = from_host([_host(m), _host(m)])
    f32 = torch.from_numpy(np.concatenate(perms).astype(np.int32)).cuda()
    i32 = torch.from_numpy(np.concatenate([np.argsort(q) for q in perms]).astype(np.int32)).cuda()
    B = ordering.permute(A, f32, i32)
    for b, q in enumerate(perms):
        o = O.permute(m, q)
        h = B.system(b)
        assert bits_equal(h.row_ptr, o.rp) and bits_equal(h.col_idx, o.ci)
        assert bits_equal(h.values, o.v)
    # vector maps (steady.py:89-94, 249-250)
    x = rng.standard_normal(m.n) + 1j * rng.standard_normal(m.n)
    xd = torch.from_numpy(x).cuda()
    q32 = torch.from_numpy(perms[0].astype(np.int32)).cuda()
    sc = ordering.permute_vector(xd, q32, 1, m.n, gather=False).cpu().numpy()
    ref = np.empty_like(x)
    ref[perms[0]] = x
    assert bits_equal(sc, ref)
    assert bits_equal(ordering.permute_vector(xd, q32, 1, m.n, gather=True).cpu().numpy(),
                      x[perms[0]])


# ---- a17: natural ordering ----------------------------------------------------
def test_c1_solve_direct_natural(cuda):
    g = G("c1")
    H, c = model("c1")
    L = liouville.build_liouvillian(H, c)
    r = steady.solve_direct(L, "natural")
    assert r.ordering == "natural" and r.method == "direct"
    assert r.residual <= 1e-10
    assert O.trace_distance(r.rho, g["direct_nat_rho"]) <= 1e-6
    assert _rel(r.fill_factor, float(g["direct_nat_fill"])) <= 1e-14
    r = steady.solve_direct(L, "rcm")
    assert O.trace_distance(r.rho, g["direct_rcm_rho"]) <= 1e-6
    assert _rel(r.fill_factor, float(g["direct_rcm_fill"])) <= 1e-14


# ---- a12: config 3 inverse power with inner GMRES(20) -------------------------
@pytest.mark.slow
def test_c3_inverse_power_gmres20(cuda):
    """BASELINE config 3: inverse power, inner GMRES(restart=20), ILUTP(1e-4,
    p=300 -- the reference default) under RCM, against the rho the reference
    produced (tests/golden/c3_gmres.npz, make_golden_r2.py --with-c3)."""
    path = os.path.join(GOLD, "c3_gmres.npz")
    if not os.path.exists(path):
        pytest.skip("c3_gmres.npz not generated")
    g = np.load(path)
    H, c = model("c3")
    L = liouville.build_liouvillian(H, c)
    r = steady.inverse_power(L, tol=1e-12, inner="iterative", ordering_name="rcm",
                             solver="gmres", restart_m=20, d=1e-4, p=300.0)
    assert r.residual <= 1e-10
    assert O.trace_distance(r.rho, g["power_gmres_rho"]) <= 1e-6
    assert r.iterations == int(g["power_gmres_iterations"])
    assert _rel(r.condest, float(g["power_gmres_condest"])) <= 1e-8
    assert _rel(r.fill_factor, float(g["power_gmres_fill"])) <= 1e-14


# ---- 'cmd' ordering where the iterate's coordinates matter --------------------
@pytest.mark.parametrize("name", ["kerr8", "c1"])
@pytest.mark.parametrize("tag,sigma", [("s3", 1e-3), ("s1", 1e-1)])
@pytest.mark.parametrize("inner", ["direct", "bicgstab"])
def test_cmd_inverse_power_large_sigma(cuda, name, tag, sigma, inner):
    """With sigma far from 0 one solve does not land on the null vector, so
    the outer iterate must stay in the original coordinates while only the
    factorization is column-ordered (steady.py:95-107, factor.py:147-148):
    same outer iteration count and steady state as the reference."""
    g = G("r2")
    H, c = configs.kerr(N=8) if name == "kerr8" else configs.kerr()
    L = liouville.build_liouvillian(H, c)
    kw = dict(sigma=sigma, tol=1e-12, ordering_name="cmd", seed=7)
    if inner == "direct":
        r = steady.inverse_power(L, inner="direct", **kw)
    else:
        r = steady.inverse_power(L, inner="iterative", solver="bicgstab", d=1e-5, p=10.0, **kw)
    key = f"{name}_cmd_{tag}_{inner}"
    assert r.ordering == str(g[key + "_label"])
    assert r.iterations == int(g[key + "_iterations"])
    assert r.residual <= 1e-10
    assert O.trace_distance(r.rho, g[key + "_rho"]) <= 1e-6
    # and the rcm path at the same shift
    if inner == "direct":
        r = steady.inverse_power(L, inner="direct", sigma=sigma, tol=1e-12,
                                 ordering_name="rcm", seed=7)
        assert r.iterations == int(g[f"{name}_rcm_{tag}_direct_iterations"])
        assert O.trace_distance(r.rho, g[f"{name}_rcm_{tag}_direct_rho"]) <= 1e-6


@pytest.mark.parametrize("solver", ["gmres", "bicgstab"])
def test_krylov_with_column_preordered_preconditioner(cuda, solver):
    """krylov.gmres / bicgstab with factor.ilutp(col_perm=...) apply the
    preconditioner with its x[q] = y scatter (krylov.py via factor.solve_lu)."""
    g = G("r2")
    H, c = model("c1")
    L = liouville.build_liouvillian(H, c)
    mod = liouville.build_modified(L, w=float(G("c1")["w"]))
    f = factor.ilutp(mod, d=1e-5, p=10.0, col_perm=Permutation(g["kry_colfwd"]))
    run = krylov.gmres if solver == "gmres" else krylov.bicgstab
    rhs = mod.rhs.cpu().numpy()
    r = run(mod, rhs, krylov.IterOptions(tol=1e-12, max_iter=200, restart_m=20,
                                         preconditioner=f))
    assert r.converged == bool(g[f"kry_{solver}_converged"])
    assert r.iterations == int(g[f"kry_{solver}_iterations"])
    ref = g[f"kry_{solver}_x"]
    assert np.linalg.norm(r.x - ref) <= 1e-10 * np.linalg.norm(ref)


def test_krylov_trace_rows(cuda):
    """trace= receives the reference's "iteration,residual" rows
    (krylov.py:62-64,152,228): same count and iteration numbers as the oracle's
    loop, residuals equal to rounding."""
    H, c = model("c1")
    L = liouville.build_liouvillian(H, c)
    mod = liouville.build_modified(L)
    fwd, inv = ordering.rcm_device(mod.matrix)
    A = ordering.permute(mod.matrix, fwd, inv)
    b = ordering.permute_vector(mod.rhs, fwd, 1, A.n, gather=False)
    f = factor.ilutp(A, d=1e-5, p=10.0)
    for run in (krylov.bicgstab, krylov.gmres):
        buf = io.StringIO()
        r = run(A, b, krylov.IterOptions(tol=1e-12, preconditioner=f), trace=buf)
        rows = [ln.split(",") for ln in buf.getvalue().splitlines()]
        its = [int(a) for a, _ in rows]
        if run is krylov.bicgstab:  # one row per loop entry, starting at iteration 0
            assert its[0] == 0 and its == sorted(its) and its[-1] in (r.iterations,
                                                                       r.iterations - 1)
        else:  # one row per Arnoldi step
            assert its == list(range(1, r.iterations + 1))
        res = [float(x) for _, x in rows]
        assert all(np.isfinite(res)) and res[-1] < res[0]


# ---- one singular system must not sink the batch ------------------------------
def test_batch_with_one_failed_factorization(cuda):
    idx = [0, 5, 9]
    mats = [liouville.build_liouvillian(*model("c4", i=i)).matrix.system(0) for i in idx]
    # system 1: column 17 of the SHIFTED matrix is exactly zero (off-diagonal
    # entries zeroed, diagonal = sigma so that L_ii - sigma = 0) -> zero pivot
    bad = mats[1]
    v = bad.values.copy()
    v[bad.col_idx == 17] = 0.0
    rows = np.repeat(np.arange(bad.nrows), np.diff(bad.row_ptr))
    hit = (bad.col_idx == 17) & (rows == 17)
    assert hit.sum() == 1
    v[hit] = liouville.DEFAULT_SIGMA
    mats[1] = CSRMatrix(bad.nrows, bad.ncols, bad.row_ptr, bad.col_idx, v)
    L = liouville.LiouvillianSystem(from_host(mats), 40, "plain")
    res = steady.inverse_power_batch(L, [2 + i for i in idx], tol=1e-12, inner="direct",
                                     ordering_name="rcm")
    assert res[1].rho is None and res[1].error.startswith("zero pivot at elimination step")
    for k in (0, 2):
        H, c = model("c4", i=idx[k])
        ref = O.inverse_power(oracle_L(H, c), 40, tol=1e-12, inner="direct", seed=2 + idx[k])
        assert res[k].error is None and res[k].residual <= 1e-10
        assert O.trace_distance(res[k].rho, ref["rho"]) <= 1e-6
    # (the trace-modified variant of system 1 keeps a 1e-15 pivot: not singular)
    out = steady.solve_batch(L, method="direct", ordering_name="rcm")
    assert out[0].error is None and out[0].residual <= 1e-10
    assert out[2].error is None and out[2].residual <= 1e-10
    with pytest.raises(ValueError):
        steady.solve_batch(L, method="cg")


# ---- seam half-solves through the C ABI ---------------------------------------
@pytest.mark.parametrize("name,kw", [("c1", {}), ("c4", {"i": 100})])
def test_half_solves_bit_exact(cuda, name, kw):
    H, c = model(name, **kw)
    Lo = oracle_L(H, c)
    m = O.build_modified(Lo, H.matrix.nrows)[0]
    fwd, _ = O.rcm(m)
    pm = O.permute(m, fwd)
    fo = O.factorize_raw(pm, 1e-5, 10.0)
    n = pm.n
    rng = np.random.default_rng(2)
    b = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    lib = O._lib()
    yl = b.copy()
    lib.orc_lower_solve(n, O._p(fo.Lp), O._p(fo.Li), O._p(fo.Lx), O._p(yl))
    yu = yl.copy()
    lib.orc_upper_solve(n, O._p(fo.Up), O._p(fo.Ui), O._p(fo.Ux), O._p(yu))

    def dev(a, dt):
        return torch.from_numpy(np.ascontiguousarray(a).astype(dt)).cuda()

    # two systems side by side (cap = entries between systems)
    for cp, ci, cx, fn, y0, ref in ((fo.Lp, fo.Li, fo.Lx, "rs_lower_solve", b, yl),
                                    (fo.Up, fo.Ui, fo.Ux, "rs_upper_solve", yl, yu)):
        cap = len(cx) + 3
        P = dev(np.concatenate([cp, cp]), np.int32)
        I = torch.zeros(2 * cap, dtype=torch.int32, device="cuda")
        X = torch.zeros(2 * cap, dtype=torch.complex128, device="cuda")
        for s in range(2):
            I[s * cap:s * cap + len(ci)] = dev(ci, np.int32)
            X[s * cap:s * cap + len(cx)] = dev(cx, np.complex128)
        y = dev(np.concatenate([y0, 2.0 * y0]), np.complex128)
        _lib.call(fn, 2, n, _lib.ptr(P), _lib.ptr(I), _lib.ptr(X), cap, _lib.ptr(y),
                  _lib.stream_ptr())
        h = y.cpu().numpy()
        assert bits_equal(h[:n], ref)
        assert np.allclose(h[n:], 2.0 * ref, rtol=1e-12, atol=0)


# ---- a1: the whole sweep assembled by one launch set ---------------------------
def test_batched_assembly_bit_exact(cuda):
    """rs_liouvillian_batch: every system of the batch bit-identical to the
    oracle's build_liouvillian (c4 instances 0 / 255 / 511 among others), also
    for members with different sparsity patterns."""
    idx = [0, 3, 255, 256, 511]
    models = [model("c4", i=i) for i in idx]
    L = liouville.build_liouvillian_batch(models)
    assert L.nsys == len(idx) and L.hilbert_dim == 40
    for b, (H, c) in enumerate(models):
        o = oracle_L(H, c)
        h = L.matrix.system(b)
        assert bits_equal(h.row_ptr, o.rp) and bits_equal(h.col_idx, o.ci)
        assert bits_equal(h.values, o.v)
    mixed = [configs.kerr(N=12), configs.kerr(N=12, chi=0.0, F=0.25), configs.kerr(N=12, delta=0.0)]
    L = liouville.build_liouvillian_batch(mixed)
    for b, (H, c) in enumerate(mixed):
        o = oracle_L(H, c)
        h = L.matrix.system(b)
        assert bits_equal(h.row_ptr, o.rp) and bits_equal(h.col_idx, o.ci)
        assert bits_equal(h.values, o.v)
    one = liouville.build_liouvillian(*mixed[1])
    assert csr_equal(one.matrix, oracle_L(*mixed[1]))
    with pytest.raises(ValueError):
        liouville.build_liouvillian_batch([configs.kerr(N=12), configs.kerr(N=10)])


# ---- the block-Jacobi opt-ins of ILUTP (NOT reference behaviour) ---------------
@pytest.mark.parametrize("early", [False, True])
def test_ilutp_optins_bit_exact_vs_oracle(cuda, early):
    """pivot_floor / early_drop (rs_factorize_opts) against the oracle carrying
    the same two opt-ins, on diagonal blocks of the RCM-ordered Kerr x Kerr
    matrix (the config-5 preconditioner) and on a block that needs the floor."""
    import scipy.sparse as sp
    H, c = configs.kerr_kerr(N=8)
    Lo = oracle_L(H, c)
    S = O.shift(Lo)
    fwd, _ = O.rcm(S)
    A = O.permute(S, fwd)
    n = A.n
    As = sp.csr_matrix((A.v, A.ci, A.rp), shape=(n, n))
    bs = n // 4
    blocks = []
    for b in range(4):
        Bk = As[b * bs:(b + 1) * bs, b * bs:(b + 1) * bs].tocsr()
        Bk.sort_indices()
        blocks.append(O.CSR(bs, bs, Bk.indptr.astype(np.int64), Bk.indices.astype(np.int64),
                            Bk.data.astype(np.complex128)))
    # block 1 gets two exactly-zero columns: one keeps stored zeros (all-zero
    # candidates), the other loses its rows to earlier pivots
    v = blocks[1].v.copy()
    v[blocks[1].ci == 5] = 0.0
    blocks[1] = O.CSR(bs, bs, blocks[1].rp, blocks[1].ci, v)
    M = from_host([_host(m) for m in blocks])
    f = factor.factor_batch(M, 1e-2, 2.0, pivot_floor=1.0, early_drop=early)
    assert f.ok
    for b, m in enumerate(blocks):
        fo = O.factorize_raw(m, 1e-2, 2.0, pivot_floor=1.0, early_drop=early)
        lp, li, lx, up, ui, ux, pinv = f.system_raw(b)
        assert bits_equal(lp, fo.Lp) and bits_equal(li, fo.Li) and bits_equal(lx, fo.Lx), b
        assert bits_equal(up, fo.Up) and bits_equal(ui, fo.Ui) and bits_equal(ux, fo.Ux), b
        assert bits_equal(pinv, fo.pinv)
        assert int(f.nfloor[b]) == fo.nfloor
    assert int(f.nfloor[1]) >= 1
    # without the floor the same block reports the reference's zero pivot
    g = factor.factor_batch(M, 1e-2, 2.0, raise_on_fail=False, early_drop=early)
    with pytest.raises(O.Breakdown) as e:
        O.factorize_raw(blocks[1], 1e-2, 2.0, early_drop=early)
    assert int(g.fail[1]) == e.value.step and g.fail[0] < 0
