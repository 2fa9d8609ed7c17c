"""Random complete-LU stress: the compact kernel against the general pipeline, bit for bit
(orders 3..400, bands 1..90, integer-valued entries for pivot ties, stored zeros, singular systems)."""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1504_06768_b200 import _lib, factor  # noqa: E402
from paper_1504_06768_b200.sparse import from_host  # noqa: E402
from tests.test_gpu_frontal import _host, _random_system  # noqa: E402

rng = np.random.default_rng(2026)
bad = 0
total = 0
for trial in range(60):
    n = int(rng.integers(3, 400))
    band = int(rng.integers(1, min(n - 1, 90) + 1))
    mats = [_random_system(rng, n, band=band, density=float(rng.uniform(0.05, 0.9)), ints=bool(k % 2))
            for k in range(int(rng.integers(1, 9)))]
    A = from_host([_host(m) for m in mats])
    os.environ["RHOSOLVE_COMPACT"] = "1"
    a = factor.factor_batch(A, 0.0, math.inf, raise_on_fail=False)
    took = _lib.load().rs_debug_compact_taken()
    os.environ["RHOSOLVE_COMPACT"] = "0"
    os.environ["RHOSOLVE_FRONTAL"] = "0"
    b = factor.factor_batch(A, 0.0, math.inf, raise_on_fail=False)
    os.environ.pop("RHOSOLVE_FRONTAL")
    same = list(a.fail) == list(b.fail)
    for s in range(len(mats)):
        if a.fail[s] >= 0:
            continue
        for x, y in zip(a.system_raw(s), b.system_raw(s)):
            same = same and x.shape == y.shape and bool(np.array_equal(x.view(np.uint8), y.view(np.uint8)))
    total += len(mats)
    if not same:
        bad += 1
        print(f"MISMATCH trial {trial}: n={n} band={band} systems={len(mats)} compact_taken={took}")
print(f"{total} systems in 60 batches, mismatching batches: {bad}")
