"""The reference's own drivers on the device kernels.

integration/install.py drops integration/_cudakernels.py into a copy of the
reference package (oracle/_ref, the unmodified reference built by
oracle/build_ref.sh) at its kernel seam (kernels/__init__.py:11-24).  The
reference's factor / krylov / steady code then runs unchanged on
rs_factorize, rs_lower_solve, rs_upper_solve and rs_csr_matvec, and must
give the SAME BITS as its compiled Cython backend: all host arithmetic
(numpy reductions, control flow) is shared, so any difference is a kernel
difference.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

from tests.helpers import bits_equal

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref")

SCRIPT = r'''
import sys
import numpy as np
sys.path.insert(0, sys.argv[2])
sys.path.insert(0, sys.argv[1])
from rhosolve import factor, kernels, krylov, liouville, operators, ordering, sparse, steady
from paper_1504_06768_b200 import configs

out = {"backend": np.array(kernels.BACKEND)}

def put(tag, r):
    out[tag + "_rho"] = r.rho
    out[tag + "_meta"] = np.array([r.residual, r.iterations, r.fill_factor,
                                   -1.0 if r.condest is None else r.condest,
                                   float(r.converged), float(r.breakdown)])

for name, (H, c), seed in (("c1", configs.kerr(ops=operators), 0),
                           ("c4", configs.jc_sweep(7, ops=operators), 9)):
    L = liouville.build_liouvillian(H, c)
    put(name + "_direct", steady.solve_direct(L, "rcm"))
    put(name + "_bicgstab", steady.solve_iterative(L, "rcm", "bicgstab", d=1e-5, p=10, tol=1e-12))
    put(name + "_gmres", steady.solve_iterative(L, "rcm", "gmres", d=1e-5, p=10, tol=1e-12))
    put(name + "_power", steady.inverse_power(L, tol=1e-12, inner="direct",
                                              ordering_name="rcm", seed=seed))
    if name == "c1":
        put(name + "_power_bicgstab",
            steady.inverse_power(L, tol=1e-12, inner="iterative", ordering_name="rcm",
                                 solver="bicgstab", d=1e-5, p=10, seed=seed))
        put(name + "_cmd", steady.solve_iterative(L, "cmd", "bicgstab", d=1e-5, p=10, tol=1e-12))
    # the four seam functions directly
    mod = liouville.build_modified(L)
    p = ordering.rcm(mod.matrix)
    m = sparse.permute(mod.matrix, p, p)
    f = factor.ilutp(m, d=1e-5, p=10.0)
    for k in ("Lp", "Li", "Lx", "Up", "Ui", "Ux"):
        out[f"{name}_f_{k}"] = getattr(f, "_" + k)
    out[name + "_f_pinv"] = f.row_perm.forward
    rng = np.random.default_rng(11)
    b = rng.standard_normal(m.nrows) + 1j * rng.standard_normal(m.nrows)
    y = b.copy()
    kernels.lower_solve(f._Lp, f._Li, f._Lx, y)
    out[name + "_lower"] = y.copy()
    kernels.upper_solve(f._Up, f._Ui, f._Ux, y)
    out[name + "_upper"] = y
    out[name + "_matvec"] = sparse.matvec(m, b)
    try:
        factor.ilutp(sparse.permute(liouville.shift(L).matrix, p, p), d=1e-5, p=10.0)
        out[name + "_fail"] = np.array(-1)
    except factor.PreconditionerBreakdownError as e:
        out[name + "_fail"] = np.array(int(str(e).rsplit(" ", 1)[-1]))
np.savez(sys.argv[3], **out)
'''


def _run(pkg_parent, backend, dest):
    env = dict(os.environ)
    env["RHOSOLVE_B200_LIB"] = os.path.join(ROOT, "paper_1504_06768_b200", "_lib",
                                            "librhosolve_b200.so")
    env["OMP_NUM_THREADS"] = env["OPENBLAS_NUM_THREADS"] = "1"
    if backend == "cuda":
        env["RHOSOLVE_BACKEND"] = "cuda"
    else:
        env.pop("RHOSOLVE_BACKEND", None)
    subprocess.run([sys.executable, "-c", SCRIPT, pkg_parent, ROOT, dest], check=True, env=env,
                   timeout=900)
    return np.load(dest)


def test_reference_drivers_on_device_kernels_bit_identical(cuda, tmp_path):
    if not os.path.isdir(os.path.join(REF, "rhosolve")):
        pytest.skip("oracle/_ref (the built reference) is not present")
    sys.path.insert(0, os.path.join(ROOT, "integration"))
    try:
        from install import install
    finally:
        sys.path.pop(0)
    install(REF, str(tmp_path))
    dev = _run(str(tmp_path), "cuda", str(tmp_path / "cuda.npz"))
    ref = _run(str(tmp_path), "c", str(tmp_path / "c.npz"))
    assert str(dev["backend"]) == "cuda" and str(ref["backend"]) == "c"
    assert set(dev.files) == set(ref.files)
    for k in ref.files:
        if k == "backend":
            continue
        assert bits_equal(dev[k], ref[k]), k
