"""SpMV on the RCM-ordered config-5 matrix (834.75 MB algorithmic): timing and
an ncu target.  python tools/spmv_c5.py [N=40] [reps=10]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1504_06768_b200 import configs, liouville, ordering  # noqa: E402
from tools.time_grid import spmv_stats  # noqa: E402


def main(N="40", reps="10"):
    L = liouville.build_liouvillian(*configs.kerr_kerr(N=int(N)))
    S = liouville.shift(L)
    fwd, inv = ordering.rcm_device(S.matrix)
    A = ordering.permute(S.matrix, fwd, inv)
    for _ in range(int(reps) // 5 + 1):
        spmv_stats(A, f"c5 N={N} rcm")
    spmv_stats(S.matrix, f"c5 N={N} natural")


if __name__ == "__main__":
    main(*sys.argv[1:])
