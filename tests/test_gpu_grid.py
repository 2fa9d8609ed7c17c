"""The grid-wide solver (csrc/grid.cu, one cooperative launch over every SM)
and its level-ordered triangular sweeps (csrc/levels.cu, csrc/trisell.cuh):
the apply bit-exact against the oracle, the solver against the reference's
steady states and iteration counts.  RHOSOLVE_GRID_MIN_N=0 routes the small
configurations through it; configs 3 and 5 take it by default."""
import os

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_1504_06768_b200 import configs, factor, liouville, sharded, steady
from paper_1504_06768_b200.sparse import CSRMatrix, from_host
from tests.helpers import bits_equal, model, oracle_L

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _host(o):
    return CSRMatrix(o.n, o.m, o.rp, o.ci, o.v)


@pytest.fixture
def grid_everything(monkeypatch):
    monkeypatch.setenv("RHOSOLVE_GRID_MIN_N", "0")
    monkeypatch.setenv("RHOSOLVE_GRID_FORCE", "1")


def _ordered(name, variant, **kw):
    H, c = model(name, **kw)
    Lo = oracle_L(H, c)
    m = O.shift(Lo) if variant == "shift" else O.build_modified(Lo, H.matrix.nrows)[0]
    fwd, _ = O.rcm(m)
    return O.permute(m, fwd)


@pytest.mark.parametrize("name,variant,d,p,kw", [
    ("c1", "shift", 1e-5, 10.0, {}), ("c1", "mod", 0.0, float("inf"), {}),
    ("c2", "mod", 1e-5, 10.0, {}), ("c2", "shift", 1e-4, 300.0, {}),
    ("c4", "mod", 1e-5, 10.0, {"i": 17})])
def test_level_sweeps_bit_exact(cuda, name, variant, d, p, kw):
    """M^{-1} b through the level-ordered sync-free sweeps == the reference
    column loops (_ckernels.pyx:53-85), bit for bit."""
    pm = _ordered(name, variant, **kw)
    fo = O.factorize_raw(pm, d, p)
    f = factor.factor_batch(from_host(_host(pm)), d, p)
    rng = np.random.default_rng(1)
    b = rng.standard_normal(pm.n) + 1j * rng.standard_normal(pm.n)
    x = factor.solve_lu_levels(f, torch.from_numpy(b).cuda()).cpu().numpy()
    assert bits_equal(x, fo.solve(b))
    assert f.Llev.nlevels >= 1 and f.Ulev.nlevels >= 1
    # the column-stream apply gives the same bits
    assert bits_equal(factor.solve_lu(f, b), x)


def test_level_sweeps_block_batch_bit_exact(cuda):
    """A batch of factors is one block-diagonal preconditioner (block-Jacobi):
    each block's rows only reach its own columns."""
    mats = [_ordered("c4", "mod", i=i) for i in (0, 200, 511)]
    f = factor.factor_batch(from_host([_host(m) for m in mats]), 1e-5, 10.0)
    n = mats[0].n
    rng = np.random.default_rng(8)
    b = rng.standard_normal(3 * n) + 1j * rng.standard_normal(3 * n)
    x = factor.solve_lu_levels(f, torch.from_numpy(b).cuda()).cpu().numpy()
    for k, m in enumerate(mats):
        assert bits_equal(x[k * n:(k + 1) * n], O.factorize_raw(m, 1e-5, 10.0).solve(b[k * n:(k + 1) * n]))


@pytest.mark.parametrize("G_rows", [(40, 0.3), (300, 0.05), (1000, 0.004)])
def test_level_sweeps_random_structures(cuda, G_rows):
    """Dense-ish, medium and very sparse random matrices: every lanes-per-row
    choice (few rows per level ... thousands of rows per level)."""
    n, dens = G_rows
    rng = np.random.default_rng(n)
    mask = rng.random((n, n)) < dens
    np.fill_diagonal(mask, True)
    r, c = np.nonzero(mask)
    v = rng.standard_normal(len(r)) + 1j * rng.standard_normal(len(r))
    v[r == c] += 4.0 * np.sqrt(n * dens)
    m = O.coo_to_csr(n, n, r, c, v, prune=False)
    fo = O.factorize_raw(m, 0.0, float("inf"))
    f = factor.factor_batch(from_host(_host(m)), 0.0, float("inf"))
    b = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    assert bits_equal(factor.solve_lu_levels(f, torch.from_numpy(b).cuda()).cpu().numpy(),
                      fo.solve(b))


def test_c1_all_methods_on_grid(cuda, grid_everything):
    g = np.load(os.path.join(GOLD, "c1.npz"))
    H, c = model("c1")
    L = liouville.build_liouvillian(H, c)
    runs = {
        "direct_rcm": lambda: steady.solve_direct(L, "rcm"),
        "bicgstab": lambda: steady.solve_iterative(L, "rcm", "bicgstab", d=1e-5, p=10, tol=1e-12),
        "gmres": lambda: steady.solve_iterative(L, "rcm", "gmres", d=1e-5, p=10, tol=1e-12),
        "power_direct": lambda: steady.inverse_power(L, tol=1e-12, inner="direct",
                                                     ordering_name="rcm", seed=0),
        "power_bicgstab": lambda: steady.inverse_power(
            L, tol=1e-12, inner="iterative", ordering_name="rcm", solver="bicgstab", d=1e-5,
            p=10, seed=0),
        "power_gmres": lambda: steady.inverse_power(
            L, tol=1e-12, inner="iterative", ordering_name="rcm", solver="gmres", d=1e-5, p=10,
            seed=0),
    }
    for key, run in runs.items():
        r = run()
        assert r.residual <= 1e-10, key
        assert O.trace_distance(r.rho, g[key + "_rho"]) <= 1e-6, key
        assert r.iterations == int(g[key + "_iterations"]), key
        if key + "_condest" in g.files:
            assert abs(r.condest - float(g[key + "_condest"])) <= 1e-10 * float(g[key + "_condest"])
    # 'cmd' ordering at a large shift: the column scatter inside the grid apply
    g2 = np.load(os.path.join(GOLD, "r2.npz"))
    r = steady.inverse_power(L, sigma=1e-1, tol=1e-12, inner="direct", ordering_name="cmd", seed=7)
    assert r.iterations == int(g2["c1_cmd_s1_direct_iterations"])
    assert O.trace_distance(r.rho, g2["c1_cmd_s1_direct_rho"]) <= 1e-6


def test_c2_on_grid(cuda, grid_everything):
    g = np.load(os.path.join(GOLD, "c2.npz"))
    H, c = model("c2")
    L = liouville.build_liouvillian(H, c)
    r = steady.inverse_power(L, tol=1e-12, inner="iterative", ordering_name="rcm",
                             solver="bicgstab", d=1e-4, p=300.0, seed=1)
    assert r.residual <= 1e-10
    assert O.trace_distance(r.rho, g["power_bicgstab_rho"]) <= 1e-6
    assert r.iterations == int(g["power_bicgstab_iterations"])
    r = steady.solve_iterative(L, "rcm", "bicgstab", d=1e-5, p=10, tol=1e-12)
    assert r.iterations == int(g["bicgstab_1e5_10_iterations"]) and r.converged
    assert O.trace_distance(r.rho, g["bicgstab_1e5_10_rho"]) <= 1e-6


def test_block_jacobi_on_grid_kerr_kerr(cuda, grid_everything):
    """Config-5 path on one GPU: RCM, block-Jacobi ILUTP (4 blocks), the whole
    inverse power in one cooperative launch; against the oracle's direct
    inverse power."""
    H, c = configs.kerr_kerr(N=10)
    L = liouville.build_liouvillian(H, c)
    res = sharded.inverse_power_sharded(L, tol=1e-10, d=1e-5, p=10.0, seed=3, blocks=4)
    ref = O.inverse_power(oracle_L(H, c), 100, tol=1e-12, inner="direct", seed=3)
    assert res.residual <= 1e-10
    assert O.trace_distance(res.rho, ref["rho"]) <= 1e-6
    assert res.extra["blocks_per_rank"] == 4


# ---- the row-sharded multi-rank driver with the real GPU ops -------------------
_RANK_SCRIPT = r'''
import os, sys
import numpy as np
import torch
import torch.distributed as dist
sys.path.insert(0, sys.argv[1])
from paper_1504_06768_b200 import configs, liouville, sharded
rank, world, port, out = int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], sys.argv[5]
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=port)
dist.init_process_group("gloo", rank=rank, world_size=world)
torch.cuda.set_device(0)  # both ranks share the one GPU; the exchange is host-staged
L = liouville.build_liouvillian(*configs.kerr_kerr(N=8))
res = sharded.inverse_power_sharded(L, tol=1e-10, d=1e-5, p=10.0, seed=3, blocks=4)
if rank == 0:
    np.savez(out, rho=res.rho, residual=res.residual, outer=res.iterations,
             inner=res.inner_iterations, world=res.extra["world"],
             blocks_per_rank=res.extra["blocks_per_rank"])
dist.destroy_process_group()
'''


def test_sharded_world2_gpu_ops(cuda, tmp_path):
    """Two ranks (gloo, host-staged halo / all-reduce, both on this GPU) run
    the row-sharded inverse power with the REAL device ops: per-rank SpMV split
    into interior and boundary rows around the halo exchange, block-Jacobi
    ILUTP factor + apply kernels, fused reductions.  Same partition as the
    one-rank grid-wide solve, so the steady states agree."""
    import socket
    import subprocess
    import sys
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = str(s.getsockname()[1])
    s.close()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = str(tmp_path / "w2.npz")
    procs = [subprocess.Popen([sys.executable, "-c", _RANK_SCRIPT, root, str(r), "2", port, out])
             for r in range(2)]
    for p in procs:
        assert p.wait(timeout=600) == 0
    w2 = np.load(out)
    assert int(w2["world"]) == 2 and int(w2["blocks_per_rank"]) == 2
    H, c = configs.kerr_kerr(N=8)
    L = liouville.build_liouvillian(H, c)
    one = sharded.inverse_power_sharded(L, tol=1e-10, d=1e-5, p=10.0, seed=3, blocks=4)
    ref = O.inverse_power(oracle_L(H, c), 64, tol=1e-12, inner="direct", seed=3)
    assert float(w2["residual"]) <= 1e-10 and one.residual <= 1e-10
    assert O.trace_distance(w2["rho"], ref["rho"]) <= 1e-6
    assert O.trace_distance(w2["rho"], one.rho) <= 1e-6
