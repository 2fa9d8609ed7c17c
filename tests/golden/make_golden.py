"""Generate the golden fixtures under tests/golden/ by running the REFERENCE
rhosolve (built into oracle/_ref by oracle/build_ref.sh, or importable from
/root/reference/pkg/src) on the BASELINE configurations.

Run in the build container (the reference does not exist on the GPU box):
    python tests/golden/make_golden.py [--with-c3]
The committed .npz files are what the CPU and GPU parity tests compare to.
Inputs (H, c_ops) come from paper_1504_06768_b200.configs with the
reference's own operator module, so both sides see the same recipe.
"""

from __future__ import annotations

import argparse
import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
for cand in (os.path.join(ROOT, "oracle", "_ref"), "/root/reference/pkg/src"):
    if os.path.isdir(os.path.join(cand, "rhosolve")):
        sys.path.insert(0, cand)
        break

import rhosolve as R  # noqa: E402
from rhosolve import factor as RF  # noqa: E402
from rhosolve import liouville as RL  # noqa: E402
from rhosolve import operators as RO  # noqa: E402
from rhosolve import ordering as ROrd  # noqa: E402
from rhosolve import sparse as RS  # noqa: E402
from rhosolve import steady as RSt  # noqa: E402

from paper_1504_06768_b200 import configs  # noqa: E402

assert R.KERNEL_BACKEND == "c", R.KERNEL_BACKEND


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def csr_arrays(prefix, m, out):
    out[prefix + "_rp"] = m.row_ptr
    out[prefix + "_ci"] = m.col_idx
    out[prefix + "_v"] = m.values


def csr_hash(m):
    return sha(m.row_ptr.astype(np.int64), m.col_idx.astype(np.int64), m.values)


def ops_arrays(H, c_ops, out):
    csr_arrays("H", H.matrix, out)
    out["n_cops"] = np.array(len(c_ops))
    for k, c in enumerate(c_ops):
        csr_arrays(f"C{k}", c.matrix, out)


def results(prefix, res, out):
    out[prefix + "_rho"] = res.rho
    out[prefix + "_residual"] = np.array(res.residual)
    out[prefix + "_iterations"] = np.array(res.iterations)
    out[prefix + "_fill"] = np.array(res.fill_factor)
    if res.condest is not None:
        out[prefix + "_condest"] = np.array(res.condest)


def common(L, D, out, full):
    sh = RL.shift(L)
    mod = RL.build_modified(L)
    p_sh = ROrd.rcm(sh.matrix)
    p_mod = ROrd.rcm(mod.matrix)
    out["D"] = np.array(D)
    out["w"] = np.array(mod.weight)
    out["rcm_shift_fwd"] = p_sh.forward
    out["rcm_shift_inv"] = p_sh.inverse
    out["rcm_mod_fwd"] = p_mod.forward
    out["rcm_mod_inv"] = p_mod.inverse
    out["L_sha"] = np.array(csr_hash(L.matrix))
    out["shift_sha"] = np.array(csr_hash(sh.matrix))
    out["mod_sha"] = np.array(csr_hash(mod.matrix))
    bp = ROrd.band_profile(RS.permute(sh.matrix, p_sh, p_sh))
    out["band_shift_rcm"] = np.array([bp.ub, bp.lb, bp.bandwidth, bp.up, bp.lp, bp.profile])
    if full:
        csr_arrays("L", L.matrix, out)
    return sh, mod, p_sh, p_mod


def kernel_outputs(prefix, mat, d, p, out, seed=42):
    """Raw factorize / solve_lu / matvec outputs of the reference kernels."""
    try:
        f = RF.ilutp(mat, d=d, p=p) if (d > 0 or np.isfinite(p)) else RF.lu(mat)
    except (RF.PreconditionerBreakdownError, RF.SingularMatrixError) as e:
        out[prefix + "_fail"] = np.array(int(str(e).rsplit(" ", 1)[-1]))
        return
    for k in ("Lp", "Li", "Lx", "Up", "Ui", "Ux"):
        out[f"{prefix}_{k}"] = getattr(f, "_" + k)
    out[prefix + "_pinv"] = f.row_perm.forward
    rng = np.random.default_rng(seed)
    b = rng.standard_normal(mat.nrows) + 1j * rng.standard_normal(mat.nrows)
    out[prefix + "_b"] = b
    out[prefix + "_solve"] = RF.solve_lu(f, b)
    out[prefix + "_matvec"] = RS.matvec(mat, b)
    out[prefix + "_condest"] = np.array(RF.condest(f))


def gen_c1():
    H, c = configs.kerr(ops=RO)
    L = RL.build_liouvillian(H, c)
    out = {}
    ops_arrays(H, c, out)
    sh, mod, p_sh, p_mod = common(L, 20, out, full=True)
    psh = RS.permute(sh.matrix, p_sh, p_sh)
    pmod = RS.permute(mod.matrix, p_mod, p_mod)
    kernel_outputs("f_sh_1e5_10", psh, 1e-5, 10.0, out)
    kernel_outputs("f_sh_lu", psh, 0.0, np.inf, out)
    kernel_outputs("f_mod_1e5_10", pmod, 1e-5, 10.0, out)
    results("direct_rcm", RSt.solve_direct(L, "rcm"), out)
    results("direct_nat", RSt.solve_direct(L, "natural"), out)
    results("bicgstab", RSt.solve_iterative(L, "rcm", "bicgstab", d=1e-5, p=10, tol=1e-12), out)
    results("gmres", RSt.solve_iterative(L, "rcm", "gmres", d=1e-5, p=10, tol=1e-12), out)
    results("power_direct", RSt.inverse_power(L, tol=1e-12, inner="direct",
                                              ordering_name="rcm", seed=0), out)
    results("power_bicgstab", RSt.inverse_power(L, tol=1e-12, inner="iterative",
                                                ordering_name="rcm", solver="bicgstab",
                                                d=1e-5, p=10, seed=0), out)
    results("power_gmres", RSt.inverse_power(L, tol=1e-12, inner="iterative",
                                             ordering_name="rcm", solver="gmres",
                                             d=1e-5, p=10, seed=0), out)
    out["start_seed0"] = RSt._start_vector(400, 0)
    return out


def gen_c2():
    H, c = configs.jc_rwa(ops=RO)
    L = RL.build_liouvillian(H, c)
    out = {}
    ops_arrays(H, c, out)
    sh, mod, p_sh, p_mod = common(L, 80, out, full=False)
    psh = RS.permute(sh.matrix, p_sh, p_sh)
    try:
        RF.ilutp(psh, d=1e-5, p=10.0)
        out["f_sh_1e5_10_fail"] = np.array(-1)
    except RF.PreconditionerBreakdownError as e:
        out["f_sh_1e5_10_fail"] = np.array(int(str(e).rsplit(" ", 1)[-1]))
    f = RF.ilutp(psh, d=1e-4, p=300.0)
    out["f_sh_def_sha"] = np.array(sha(f._Lp, f._Li, f._Lx, f._Up, f._Ui, f._Ux))
    out["f_sh_def_nnz"] = np.array([len(f._Lx), len(f._Ux)])
    results("power_bicgstab", RSt.inverse_power(L, tol=1e-12, inner="iterative",
                                                ordering_name="rcm", solver="bicgstab",
                                                d=1e-4, p=300.0, seed=1), out)
    results("power_direct", RSt.inverse_power(L, tol=1e-12, inner="direct",
                                              ordering_name="rcm", seed=1), out)
    results("bicgstab_1e5_10", RSt.solve_iterative(L, "rcm", "bicgstab", d=1e-5, p=10,
                                                   tol=1e-12), out)
    return out


def gen_c4():
    out = {}
    dets = configs.jc_sweep_detunings()
    out["detunings"] = dets
    for i in (0, 255, 511):
        H, c = configs.jc_sweep(i, ops=RO)
        L = RL.build_liouvillian(H, c)
        sub = {}
        common(L, 40, sub, full=(i == 0))
        if i == 0:
            ops_arrays(H, c, sub)
        res = RSt.inverse_power(L, tol=1e-12, inner="direct", ordering_name="rcm", seed=2 + i)
        results("power_direct", res, sub)
        res = RSt.solve_iterative(L, "rcm", "bicgstab", d=1e-5, p=10, tol=1e-12)
        results("bicgstab_1e5_10", res, sub)
        for k, v in sub.items():
            out[f"i{i}_{k}"] = v
    return out


def gen_c3():
    H, c = configs.optomech(ops=RO)
    L = RL.build_liouvillian(H, c)
    out = {}
    sh, mod, p_sh, p_mod = common(L, 240, out, full=False)
    t = time.time()
    res = RSt.inverse_power(L, tol=1e-12, inner="iterative", ordering_name="rcm",
                            solver="bicgstab", d=1e-4, p=300.0)
    out["power_bicgstab_wall"] = np.array(time.time() - t)
    results("power_bicgstab", res, out)
    return out


def gen_rcm_corpus():
    """Seeded random structures (own generator) and the reference RCM."""
    rng = np.random.default_rng(20261020)
    out = {}
    for k in range(30):
        n = int(rng.integers(2, 60))
        dens = float(rng.uniform(0.02, 0.3))
        mask = rng.random((n, n)) < dens
        if k % 3 == 0:  # force some isolated nodes / several components
            mask[:, : n // 3] = False
            mask[: n // 3, :] = False
        r, cidx = np.nonzero(mask)
        m = RS.SparseComplexMatrix.from_coo(n, n, r, cidx, np.ones(len(r)))
        p = ROrd.rcm(m)
        out[f"s{k}_n"] = np.array(n)
        out[f"s{k}_rp"] = m.row_ptr
        out[f"s{k}_ci"] = m.col_idx
        out[f"s{k}_inv"] = p.inverse
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--with-c3", action="store_true")
    args = ap.parse_args()
    jobs = [("c1", gen_c1), ("c2", gen_c2), ("c4", gen_c4), ("rcm_corpus", gen_rcm_corpus)]
    if args.with_c3:
        jobs.append(("c3", gen_c3))
    for name, fn in jobs:
        t = time.time()
        out = fn()
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
        print(f"{name}: {len(out)} arrays in {time.time() - t:.1f}s")


if __name__ == "__main__":
    main()
