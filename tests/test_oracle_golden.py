"""Pin the CPU oracle to the reference: every golden vector in tests/golden
was produced by the reference rhosolve itself (tests/golden/make_golden.py).
Bit-exact for structure/index/kernel outputs; tolerance for Krylov-level
results (numpy BLAS reduction order)."""
import hashlib
import math
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests.helpers import bits_equal, model

G = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    return np.load(os.path.join(G, f"{name}.npz"))


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def csr_sha(m):
    return sha(m.rp.astype(np.int64), m.ci.astype(np.int64), m.v)


def test_c1_assembly_and_variants():
    g = load("c1")
    H, c = model("c1")
    L = O.build_liouvillian(H.matrix, [x.matrix for x in c])
    assert bits_equal(L.rp, g["L_rp"]) and bits_equal(L.ci, g["L_ci"])
    assert bits_equal(L.v, g["L_v"])
    assert csr_sha(L) == str(g["L_sha"])
    assert csr_sha(O.shift(L)) == str(g["shift_sha"])
    w = O.default_weight(L)
    assert w == float(g["w"])
    assert csr_sha(O.build_modified(L, 20, w)[0]) == str(g["mod_sha"])


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_rcm_matches_reference(name):
    g = load(name)
    H, c = model(name)
    L = O.build_liouvillian(H.matrix, [x.matrix for x in c])
    assert csr_sha(L) == str(g["L_sha"])
    fwd, inv = O.rcm(O.shift(L))
    assert bits_equal(fwd, g["rcm_shift_fwd"]) and bits_equal(inv, g["rcm_shift_inv"])
    fwd, inv = O.rcm(O.build_modified(L, int(g["D"]))[0])
    assert bits_equal(fwd, g["rcm_mod_fwd"]) and bits_equal(inv, g["rcm_mod_inv"])


def test_rcm_random_corpus():
    g = load("rcm_corpus")
    k = 0
    while f"s{k}_n" in g:
        n = int(g[f"s{k}_n"])
        A = O.CSR(n, n, g[f"s{k}_rp"], g[f"s{k}_ci"], np.ones(len(g[f"s{k}_ci"])))
        _, inv = O.rcm(A)
        assert bits_equal(inv, g[f"s{k}_inv"]), k
        k += 1
    assert k == 30


@pytest.mark.parametrize("prefix,variant,d,p", [
    ("f_sh_1e5_10", "shift", 1e-5, 10.0), ("f_sh_lu", "shift", 0.0, math.inf),
    ("f_mod_1e5_10", "mod", 1e-5, 10.0)])
def test_c1_kernels_bit_exact(prefix, variant, d, p):
    g = load("c1")
    H, c = model("c1")
    L = O.build_liouvillian(H.matrix, [x.matrix for x in c])
    m = O.shift(L) if variant == "shift" else O.build_modified(L, 20)[0]
    fwd = g[f"rcm_{'shift' if variant == 'shift' else 'mod'}_fwd"]
    pm = O.permute(m, fwd)
    f = O.factorize_raw(pm, d, p)
    for k in ("Lp", "Li", "Lx", "Up", "Ui", "Ux"):
        assert bits_equal(getattr(f, k), g[f"{prefix}_{k}"]), k
    assert bits_equal(f.pinv, g[f"{prefix}_pinv"])
    b = g[f"{prefix}_b"]
    assert bits_equal(f.solve(b), g[f"{prefix}_solve"])
    assert bits_equal(O.csr_matvec(pm, b), g[f"{prefix}_matvec"])
    assert O.condest(f) == float(g[f"{prefix}_condest"])


def test_c2_factor_and_breakdown():
    g = load("c2")
    H, c = model("c2")
    L = O.shift(O.build_liouvillian(H.matrix, [x.matrix for x in c]))
    pm = O.permute(L, g["rcm_shift_fwd"])
    with pytest.raises(O.Breakdown) as e:
        O.factorize_raw(pm, 1e-5, 10.0)
    assert e.value.step == int(g["f_sh_1e5_10_fail"])
    f = O.factorize_raw(pm, 1e-4, 300.0)
    assert sha(f.Lp, f.Li, f.Lx, f.Up, f.Ui, f.Ux) == str(g["f_sh_def_sha"])


def test_c1_solutions_match_reference():
    g = load("c1")
    H, c = model("c1")
    L = O.build_liouvillian(H.matrix, [x.matrix for x in c])
    ip = O.inverse_power(L, 20, tol=1e-12, inner="iterative", solver="bicgstab", d=1e-5,
                         p=10, seed=0)
    assert O.trace_distance(ip["rho"], g["power_bicgstab_rho"]) <= 1e-12
    assert ip["outer"] == int(g["power_bicgstab_iterations"])
    ip = O.inverse_power(L, 20, tol=1e-12, inner="direct", seed=0)
    assert O.trace_distance(ip["rho"], g["power_direct_rho"]) <= 1e-12
    lin = O.solve_linear(L, 20, "bicgstab", d=1e-5, p=10, tol=1e-12)
    assert O.trace_distance(lin["rho"], g["bicgstab_rho"]) <= 1e-12
    assert lin["iterations"] == int(g["bicgstab_iterations"])
    lin = O.solve_linear(L, 20, "direct")
    assert O.trace_distance(lin["rho"], g["direct_rcm_rho"]) <= 1e-12
    assert bits_equal(O.start_vector(400, 0), g["start_seed0"])


def test_c4_sweep_rcm_and_rho():
    g = load("c4")
    for i in (0, 255, 511):
        H, c = model("c4", i=i)
        L = O.build_liouvillian(H.matrix, [x.matrix for x in c])
        assert csr_sha(L) == str(g[f"i{i}_L_sha"])
        fwd, _ = O.rcm(O.shift(L))
        assert bits_equal(fwd, g[f"i{i}_rcm_shift_fwd"])
    # structure and RCM identical across the sweep
    assert bits_equal(g["i0_rcm_shift_fwd"], g["i511_rcm_shift_fwd"])
    H, c = model("c4", i=0)
    L = O.build_liouvillian(H.matrix, [x.matrix for x in c])
    ip = O.inverse_power(L, 40, tol=1e-12, inner="direct", seed=2)
    assert O.trace_distance(ip["rho"], g["i0_power_direct_rho"]) <= 1e-12


def test_c2_c3_reference_results_are_physical():
    for name in ("c2", "c3"):
        g = load(name)
        rho = g["power_bicgstab_rho"]
        assert float(g["power_bicgstab_residual"]) <= 1e-10
        assert abs(np.trace(rho) - 1) < 1e-12
        assert np.max(np.abs(rho - rho.conj().T)) < 1e-12


@pytest.mark.parametrize("name,kw", [("c1", {}), ("c2", {}), ("c4", {"i": 0}), ("c4", {"i": 511})])
def test_rcm_of_plain_equals_rcm_of_shifted(name, kw):
    """The GPU path orders the plain pattern while the shifted values are
    still uploading (steady._power_core): valid because the RCM graph drops
    self-loops (ordering.py:62-79) and shifting only adds diagonal entries."""
    H, c = model(name, **kw)
    Lo = O.build_liouvillian(H.matrix, [x.matrix for x in c])
    fp, ip = O.rcm(Lo)
    fs, is_ = O.rcm(O.shift(Lo))
    assert bits_equal(fp, fs) and bits_equal(ip, is_)
