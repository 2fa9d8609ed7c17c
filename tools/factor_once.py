"""Run one factorization of a configuration (for ncu captures)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1504_06768_b200 import configs, factor, liouville, ordering  # noqa: E402


def main(cfg="c2", count="1"):
    c = configs.CONFIGS[cfg]
    if cfg == "c4":
        L = liouville.build_liouvillian_batch([configs.jc_sweep(i) for i in range(int(count))])
        d, p = 0.0, float("inf")
    else:
        L = liouville.build_liouvillian(*c["build"]())
        d, p = c["d"], c["p"]
    sh = liouville.shift(L)
    fwd, inv = ordering.rcm_device(sh.matrix)
    A = ordering.permute(sh.matrix, fwd, inv)
    f = factor.factor_batch(A, d, p)
    torch.cuda.synchronize()
    print("ok", f.fill_factors[:4])


if __name__ == "__main__":
    main(*sys.argv[1:])
