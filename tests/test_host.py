"""Host-side logic (no GPU): operator inputs bit-identical to the reference's,
the C-ABI library loads and exports every declared symbol, API argument
checks raise the reference's errors before any device work."""
import os
import re

import numpy as np
import pytest

from paper_1504_06768_b200 import _lib, configs, liouville, sparse, steady
from tests.helpers import bits_equal

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "tests", "golden")


@pytest.mark.parametrize("name,kw", [("c1", {}), ("c2", {}), ("c4", {"i": 0})])
def test_operator_inputs_match_reference(name, kw):
    g = np.load(os.path.join(G, f"{name}.npz"))
    pre = "i0_" if name == "c4" else ""
    H, c = (configs.jc_sweep(0) if name == "c4" else configs.CONFIGS[name]["build"]())
    assert bits_equal(H.matrix.row_ptr, g[pre + "H_rp"])
    assert bits_equal(H.matrix.col_idx, g[pre + "H_ci"])
    assert bits_equal(H.matrix.values, g[pre + "H_v"])
    assert len(c) == int(g[pre + "n_cops"])
    for k, op in enumerate(c):
        assert bits_equal(op.matrix.values, g[f"{pre}C{k}_v"])
        assert bits_equal(op.matrix.col_idx, g[f"{pre}C{k}_ci"])


def test_header_symbols_exported():
    with open(os.path.join(ROOT, "include", "rhosolve_b200.h")) as fh:
        hdr = fh.read()
    declared = set(re.findall(r"^\s*(?:int|int64_t|const char\*|long long)\s+(rs_\w+)\s*\(", hdr, re.M))
    assert declared, "no declarations parsed"
    lib = _lib.load()
    for sym in sorted(declared):
        assert hasattr(lib, sym), sym
    assert set(_lib.EXPORTED) == declared
    assert lib.rs_abi_version() == 2


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    H, c = configs.kerr()
    with pytest.raises(RuntimeError, match="CUDA"):
        liouville.build_liouvillian(H, c)


def test_start_vector_is_numpy_pcg64():
    x = steady.start_vector(5, 0)
    rng = np.random.default_rng(0)
    ref = rng.standard_normal(5) + 1j * rng.standard_normal(5)
    assert bits_equal(x, ref)


def test_permutation_from_order():
    p = sparse.Permutation.from_order([2, 0, 1])
    assert list(p.forward) == [1, 2, 0] and list(p.inverse) == [2, 0, 1]


def test_jc_sweep_detunings():
    d = configs.jc_sweep_detunings()
    assert len(d) == 512 and d[0] == -3.0 and d[-1] == 3.0 and not np.any(d == 0.0)


@pytest.mark.parametrize("m", [1, 5, 100])
def test_batch_start_vectors_match_reference_draw(m):
    """The batched draw (one standard_normal(2n) per seed, two threads for
    large batches) gives the reference's start_vector bits (steady.py:171-174)."""
    seeds = list(range(2, 2 + m))
    got = steady._start_vectors(1600, seeds, pin=False).numpy()
    ref = np.concatenate([steady.start_vector(1600, s) for s in seeds])
    assert bits_equal(got, ref)


def test_bench_c4_shards_cover_the_sweep():
    """bench.py's instance sharding (config 4): contiguous, disjoint, complete
    for every world size the driver uses, detunings and seeds kept."""
    import bench
    for world in (1, 2, 4, 8):
        parts = [list(bench.shard(r, world)) for r in range(world)]
        assert sum(parts, []) == list(range(bench.SWEEP))
        assert {len(p) for p in parts} == {bench.SWEEP // world}
    idx, models = bench.build_inputs("c4", rank=1, world=2)
    assert idx[0] == 256 and len(models) == 256
    dets = configs.jc_sweep_detunings()
    H, _ = models[0]
    H0, _ = configs.jc_sweep(256)
    assert bits_equal(H.matrix.values, H0.matrix.values)
    assert dets[256] == np.linspace(-3.0, 3.0, 512)[256]
