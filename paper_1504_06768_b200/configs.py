"""The five BASELINE.json configurations as (H, c_ops) recipes.

Each builder takes an `ops` namespace providing destroy / spin_ops / embed
(default: this package's operators; the golden generator passes the
reference's `rhosolve.operators` so both sides build the *same* CSR arrays).
Construction orders are pinned because the tensor
factor order changes the RCM permutation.
"""

from __future__ import annotations

import numpy as np

from . import operators as _ops

__all__ = ["kerr", "jc_rwa", "optomech", "jc_sweep_detunings", "kerr_kerr", "CONFIGS"]


def kerr(N=20, delta=-1.0, chi=0.5, F=1.0, kappa=1.0, n_th=0.1, ops=_ops):
    """c1: driven damped Kerr oscillator, dims (N,)."""
    a = ops.destroy(N)
    ad = a.adjoint()
    H = delta * (ad @ a) + chi * (ad @ ad @ a @ a) + F * (a + ad)
    c_ops = [np.sqrt(kappa) * a, np.sqrt(kappa * n_th) * ad]
    return H, c_ops


def jc_rwa(N=40, dc=0.0, dq=0.0, g=1.0, E=0.5, kappa=0.5, gamma=0.1, ops=_ops):
    """c2 / c4: driven RWA Jaynes-Cummings, dims (N, 2) -- cavity first."""
    dims = (N, 2)
    a = ops.embed(ops.destroy(N), dims, 0)
    sm = ops.embed(ops.spin_ops()["sigma_minus"], dims, 1)
    sp = sm.adjoint()
    ad = a.adjoint()
    H = dc * (ad @ a) + dq * (sp @ sm) + g * (ad @ sm + a @ sp) + E * (a + ad)
    c_ops = [np.sqrt(kappa) * a, np.sqrt(gamma) * sm]
    return H, c_ops


def optomech(n_c=6, n_m=40, delta=-1.0, omega_m=1.0, g0=0.1, drive=0.5, kappa=0.2,
             gamma=1e-3, n_th=1.0, ops=_ops):
    """c3: optomechanics, dims (n_c, n_m) -- the reference build_optomech
    (pkg/src/rhosolve/models.py:165-192) with the config-3 overrides."""
    dims = (n_c, n_m)
    a = ops.embed(ops.destroy(n_c), dims, 0)
    b = ops.embed(ops.destroy(n_m), dims, 1)
    ad = a.adjoint()
    bd = b.adjoint()
    H = ((-delta) * (ad @ a) + omega_m * (bd @ b) + g0 * ((b + bd) @ (ad @ a))
         + drive * (a + ad))
    c_ops = [np.sqrt(kappa) * a, np.sqrt(gamma * (1.0 + n_th)) * b,
             np.sqrt(gamma * n_th) * bd]
    return H, c_ops


def jc_sweep_detunings(count=512):
    """c4 cavity detunings: np.linspace(-3, 3, 512)."""
    return np.linspace(-3.0, 3.0, count)


def jc_sweep(i, N=20, count=512, ops=_ops):
    """c4 instance i: N=20 cavity x qubit, E=0.3, detuning dc_i, seed 2+i."""
    return jc_rwa(N=N, dc=float(jc_sweep_detunings(count)[i]), dq=0.0, g=1.0, E=0.3,
                  kappa=0.5, gamma=0.1, ops=ops)


def kerr_kerr(N=40, delta=-0.5, chi=0.2, F=0.8, J=0.5, kappa=1.0, ops=_ops):
    """c5: two coupled driven Kerr cavities, dims (N, N)."""
    dims = (N, N)
    a1 = ops.embed(ops.destroy(N), dims, 0)
    a2 = ops.embed(ops.destroy(N), dims, 1)
    terms = None
    for a in (a1, a2):
        ad = a.adjoint()
        t = delta * (ad @ a) + chi * (ad @ ad @ a @ a) + F * (a + ad)
        terms = t if terms is None else terms + t
    H = terms + J * (a1.adjoint() @ a2 + a2.adjoint() @ a1)
    c_ops = [np.sqrt(kappa) * a1, np.sqrt(kappa) * a2]
    return H, c_ops


# Solver settings per configuration (BASELINE.json "configs").
CONFIGS = {
    "c1": dict(build=kerr, D=20, tol=1e-12, seed=0, d=1e-5, p=10.0,
               methods=("direct", "bicgstab", "power-direct", "power-bicgstab")),
    "c2": dict(build=jc_rwa, D=80, tol=1e-12, seed=1, d=1e-4, p=300.0,
               methods=("bicgstab", "power-bicgstab", "power-direct")),
    "c3": dict(build=optomech, D=240, tol=1e-12, seed=12345, d=1e-4, p=300.0,
               methods=("power-gmres", "power-bicgstab")),
    "c4": dict(build=jc_sweep, D=40, tol=1e-12, seed=2, d=1e-5, p=10.0,
               methods=("power-direct",)),
    # block-Jacobi ILUTP over 40 RCM row blocks with the two opt-ins of
    # rs_factorize_opts (config 5): the reference names no (d, p) here
    "c5": dict(build=kerr_kerr, D=1600, tol=1e-10, seed=3, d=1e-2, p=2.0, blocks=40,
               pivot_floor=1.0, early_drop=True, methods=("power-bicgstab",)),
}
