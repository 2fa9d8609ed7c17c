"""Per-stage CUDA-event breakdown of one inverse-power solve (single system or
batch) through the public API pieces, for tuning."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1504_06768_b200 import _lib, configs, factor, liouville, ordering, steady  # noqa: E402


class Timer:
    def __init__(self):
        self.marks = []

    def mark(self, name):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        self.marks.append((name, e, time.perf_counter()))

    def report(self):
        torch.cuda.synchronize()
        for (n0, e0, h0), (n1, e1, h1) in zip(self.marks, self.marks[1:]):
            print(f"  {n1:14s} gpu {e0.elapsed_time(e1):9.2f} ms   host {1e3 * (h1 - h0):9.2f} ms")


def main(cfg="c4", count="512"):
    c = configs.CONFIGS[cfg]
    if cfg == "c4":
        models = [configs.jc_sweep(i) for i in range(int(count))]
        L = liouville.build_liouvillian_batch(models)
        seeds = [2 + i for i in range(len(models))]
        d, p, inner = 0.0, float("inf"), "direct"
    else:
        L = liouville.build_liouvillian(*c["build"]())
        seeds = [c["seed"]]
        d, p, inner = c["d"], c["p"], "iterative"
    for rep in range(3):
        T = Timer()
        torch.cuda.synchronize()
        T.mark("start")
        sh = liouville.shift(L)
        T.mark("shift")
        fwd, inv = ordering.rcm_device(sh.matrix)
        T.mark("rcm")
        A = ordering.permute(sh.matrix, fwd, inv)
        P = ordering.permute(L.matrix, fwd, inv)
        T.mark("permute x2")
        f = factor.factor_batch(A, d, p)
        T.mark("factor")
        x0 = torch.from_numpy(np.concatenate([steady.start_vector(A.n, s) for s in seeds])).cuda()
        T.mark("start vec")
        mode = _lib.INV_DIRECT if inner == "direct" else _lib.INV_BICGSTAB
        x, st = steady._solve(mode, A, P, f, x0, c["tol"], 1000, 20, inner != "direct")
        T.mark("solver")
        rho, res = steady._postprocess(x, fwd, L)
        T.mark("postprocess")
        if rep == 2:
            print(cfg, "systems", L.nsys, "n", L.n, "fill", float(np.mean(f.fill_factors)))
            T.report()


if __name__ == "__main__":
    main(*sys.argv[1:])
