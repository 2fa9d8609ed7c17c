"""Interchange formats and the sweep record schema
against fixtures written by the reference itself (tests/golden/io, made by
tests/golden/make_golden_io.py): Matrix Market writer bytes and reader
arrays, Permutation save/load, BenchRecord CSV bytes and round trip."""
import dataclasses
import math
import os

import numpy as np
import pytest

from paper_1504_06768_b200 import sparse, sweep
from paper_1504_06768_b200.sparse import CSRMatrix, Permutation

IO = os.path.join(os.path.dirname(__file__), "golden", "io")


def _random_matrix():
    # the same recipe as make_golden_io.random_matrix (numpy RNG, our from_coo)
    rng = np.random.default_rng(1504)
    r = rng.integers(0, 12, 40)
    c = rng.integers(0, 9, 40)
    v = rng.standard_normal(40) + 1j * rng.standard_normal(40)
    v[0] = complex(-0.0, 0.0)
    v[1] = complex(5e-324, -1e300)
    v[2] = complex(1.0 / 3.0, -2.0 / 3.0)
    v[3] = complex(0.0, -0.0)
    return CSRMatrix.from_coo(12, 9, r, c, v, prune=False)


def _read(name):
    with open(os.path.join(IO, name), "rb") as fh:
        return fh.read()


def test_matrix_market_writer_bytes(tmp_path):
    out = tmp_path / "m.mtx"
    sparse.write_matrix_market(_random_matrix(), out, comment="rhosolve golden\nsecond line")
    assert out.read_bytes() == _read("mm_random.mtx")


def test_matrix_market_round_trip(tmp_path):
    m = _random_matrix()
    back = sparse.read_matrix_market(os.path.join(IO, "mm_random.mtx"))
    assert back.shape == m.shape
    assert np.array_equal(back.row_ptr, m.row_ptr) and np.array_equal(back.col_idx, m.col_idx)
    assert np.array_equal(back.values.view(np.float64), m.values.view(np.float64))


def test_matrix_market_reader_real_duplicates():
    m = sparse.read_matrix_market(os.path.join(IO, "mm_mixed_in.mtx"))
    ref = np.load(os.path.join(IO, "mm_mixed_read.npz"))
    assert tuple(ref["shape"]) == m.shape
    assert np.array_equal(m.row_ptr, ref["rp"]) and np.array_equal(m.col_idx, ref["ci"])
    assert np.array_equal(m.values.view(np.float64), ref["v"].view(np.float64))


@pytest.mark.parametrize("text,err", [
    ("%%MatrixMarket matrix array complex general\n1 1\n", "header"),
    ("%%MatrixMarket matrix coordinate complex symmetric\n1 1 0\n", "symmetry"),
    ("%%MatrixMarket matrix coordinate pattern general\n1 1 0\n", "field type"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n", "expected 2"),
])
def test_matrix_market_reader_errors(tmp_path, text, err):
    p = tmp_path / "bad.mtx"
    p.write_text(text)
    with pytest.raises(ValueError, match=err):
        sparse.read_matrix_market(p)


def test_permutation_save_load(tmp_path):
    p = Permutation.from_order(np.array([3, 0, 4, 1, 2]))
    out = tmp_path / "p.txt"
    p.save(out)
    assert out.read_bytes() == _read("perm.txt")
    q = Permutation.load(out)
    assert np.array_equal(q.forward, p.forward) and np.array_equal(q.inverse, p.inverse)
    with pytest.raises(ValueError, match="bijection"):
        Permutation(np.array([0, 0, 1]))


def _records():
    common = dict(system="kerr", size=20, hilbert_dim=20, liouvillian_variant="modified",
                  nnz_L_liouvillian=2660, bandwidth_before=41, bandwidth_after=43,
                  bandwidth_reduction=41 / 43, profile_before=1234, profile_after=567,
                  profile_reduction=1234 / 567, d=1e-5, p=10.0, tol=1e-12, m=20, sigma=1e-15,
                  w=0.7142857142857143, seed=0)
    return [sweep.BenchRecord(ordering="rcm", method="iterative-bicgstab", fill_factor=3.03125,
                              condest=14.123456789012345, converged=True, breakdown=False,
                              iterations=2, residual=4.1e-15, build_time=0.001,
                              factor_time=0.0123, solve_time=1.0 / 3.0, **common),
            sweep.BenchRecord(ordering="cmd", method="gmres", fill_factor=float("nan"),
                              condest=None, converged=False, breakdown=True, iterations=0,
                              residual=float("nan"), build_time=0.0, factor_time=0.0,
                              solve_time=2.5e-7, **common)]


def test_records_csv_bytes_and_round_trip(tmp_path):
    out = tmp_path / "r.csv"
    recs = _records()
    sweep.write_results(recs, out)
    assert out.read_bytes() == _read("records.csv")
    back = sweep.read_results(out)
    assert len(back) == 2
    for a, b in zip(recs, back):
        for f in dataclasses.fields(a):
            x, y = getattr(a, f.name), getattr(b, f.name)
            if f.name.endswith("_reduction"):
                assert y == float(f"{x:.4g}")
            elif isinstance(x, float) and math.isnan(x):
                assert math.isnan(y)
            else:
                assert x == y, f.name
    sweep.write_results(recs, tmp_path / "r.json", fmt="json")
    with pytest.raises(ValueError):
        sweep.write_results(recs, tmp_path / "r.x", fmt="xml")


def test_sweep_spec_checks():
    with pytest.raises(ValueError, match="unknown method"):
        sweep.SweepSpec("kerr", [4], ["nope"], ["rcm"]).check()
    with pytest.raises(ValueError, match="unknown ordering"):
        sweep.SweepSpec("kerr", [4], ["direct"], ["amd"]).check()
    with pytest.raises(ValueError, match="sizes"):
        sweep.SweepSpec("kerr", [1], ["direct"], ["rcm"]).check()
    with pytest.raises(ValueError, match="unknown system"):
        sweep.SweepSpec("spin_chain", [4], ["direct"], ["rcm"]).check()
    sweep.SweepSpec("kerr", [4], list(sweep.METHODS), list(sweep.ORDERINGS)).check()
