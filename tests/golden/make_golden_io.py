"""Golden fixtures for the interchange / reporting rows (SURVEY.md 8(f) f3,
f4), written by the REFERENCE rhosolve itself:
  io/mm_random.mtx       write_matrix_market of a small matrix with special
                         values (signed zeros, subnormal, huge, thirds)
  io/mm_mixed_in.mtx     a hand-made real-valued input with duplicates and
                         comments; io/mm_mixed_read.npz = the reference
                         reader's CSR of it
  io/perm.txt            Permutation.save of a fixed permutation
  io/records.csv         write_results of two BenchRecords (one failed)
  io/export_c1.json      sha256 of export_factors' four files for the c1
                         shifted RCM-ordered complete LU
Run in the build container: python tests/golden/make_golden_io.py
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "io")
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
for cand in (os.path.join(ROOT, "oracle", "_ref"), "/root/reference/pkg/src"):
    if os.path.isdir(os.path.join(cand, "rhosolve")):
        sys.path.insert(0, cand)
        break

from rhosolve import bench as RB  # noqa: E402
from rhosolve import factor as RF  # noqa: E402
from rhosolve import liouville as RL  # noqa: E402
from rhosolve import operators as RO  # noqa: E402
from rhosolve import ordering as ROrd  # noqa: E402
from rhosolve import sparse as RS  # noqa: E402

from paper_1504_06768_b200 import configs  # noqa: E402


def random_matrix():
    rng = np.random.default_rng(1504)
    r = rng.integers(0, 12, 40)
    c = rng.integers(0, 9, 40)
    v = rng.standard_normal(40) + 1j * rng.standard_normal(40)
    v[0] = complex(-0.0, 0.0)
    v[1] = complex(5e-324, -1e300)
    v[2] = complex(1.0 / 3.0, -2.0 / 3.0)
    v[3] = complex(0.0, -0.0)
    return RS.SparseComplexMatrix.from_coo(12, 9, r, c, v, prune=False)


MIXED = """%%MatrixMarket matrix coordinate real general
% comment line
%
4 5 6
1 1 1.5
2 3 -2
1 1 0.25

4 5 1e-3
3 2 7
2 3 2
"""


def sha_file(path):
    with open(path, "rb") as fh:
        return hashlib.sha256(fh.read()).hexdigest()


def main():
    os.makedirs(OUT, exist_ok=True)
    RS.write_matrix_market(random_matrix(), os.path.join(OUT, "mm_random.mtx"),
                           comment="rhosolve golden\nsecond line")
    with open(os.path.join(OUT, "mm_mixed_in.mtx"), "w") as fh:
        fh.write(MIXED)
    m = RS.read_matrix_market(os.path.join(OUT, "mm_mixed_in.mtx"))
    np.savez(os.path.join(OUT, "mm_mixed_read.npz"), rp=m.row_ptr, ci=m.col_idx, v=m.values,
             shape=np.array([m.nrows, m.ncols]))
    RS.Permutation.from_order(np.array([3, 0, 4, 1, 2])).save(os.path.join(OUT, "perm.txt"))

    common = dict(system="kerr", size=20, hilbert_dim=20, liouvillian_variant="modified",
                  nnz_L_liouvillian=2660, bandwidth_before=41, bandwidth_after=43,
                  bandwidth_reduction=41 / 43, profile_before=1234, profile_after=567,
                  profile_reduction=1234 / 567, d=1e-5, p=10.0, tol=1e-12, m=20, sigma=1e-15,
                  w=0.7142857142857143, seed=0)
    recs = [RB.BenchRecord(ordering="rcm", method="iterative-bicgstab", fill_factor=3.03125,
                           condest=14.123456789012345, converged=True, breakdown=False,
                           iterations=2, residual=4.1e-15, build_time=0.001,
                           factor_time=0.0123, solve_time=1.0 / 3.0, **common),
            RB.BenchRecord(ordering="cmd", method="gmres", fill_factor=float("nan"),
                           condest=None, converged=False, breakdown=True, iterations=0,
                           residual=float("nan"), build_time=0.0, factor_time=0.0,
                           solve_time=2.5e-7, **common)]
    RB.write_results(recs, os.path.join(OUT, "records.csv"))

    H, c = configs.kerr(ops=RO)
    L = RL.build_liouvillian(H, c)
    sh = RL.shift(L).matrix
    p = ROrd.rcm(sh)
    A = RS.permute(sh, p, p)
    f = RF.lu(A)
    with tempfile.TemporaryDirectory() as td:
        pre = os.path.join(td, "c1")
        RF.export_factors(f, pre)
        hashes = {k: sha_file(f"{pre}{k}") for k in ("_L.mtx", "_U.mtx", "_rowperm.txt",
                                                      "_colperm.txt")}
    with open(os.path.join(OUT, "export_c1.json"), "w") as fh:
        json.dump(hashes, fh, indent=1)
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
