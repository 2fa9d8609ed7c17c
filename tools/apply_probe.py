"""Preconditioner apply M^{-1} b: column sweeps on the raw CSC factors
(colsweep.cuh) vs the row-oriented warp-per-row sweeps, bit-compared and
event-timed (tuning)."""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1504_06768_b200 import configs, factor, liouville, ordering  # noqa: E402


def timed(fn, reps=5):
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        flush.zero_()
        torch.cuda._sleep(100_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts[1:])


def main(cfg, count=1):
    if cfg == "c4":
        L = liouville.build_liouvillian_batch([configs.jc_sweep(i) for i in range(count)])
        d, p = 0.0, math.inf
    else:
        c = configs.CONFIGS[cfg]
        L = liouville.build_liouvillian(*c["build"]())
        d, p = c["d"], c["p"]
    sh = liouville.shift(L)
    fwd, inv = ordering.rcm_device(sh.matrix)
    A = ordering.permute(sh.matrix, fwd, inv)
    f = factor.factor_batch(A, d, p)
    x = torch.randn(A.n * A.nsys, dtype=torch.complex128, device="cuda")
    nLU = int(sum(f.lnnz) + sum(f.unnz))
    byt = 20 * nLU + 72 * A.n * A.nsys
    out = {}
    for csc in (True, False):
        f.csc = csc
        if not csc:
            f.ensure_rows()
        out[csc] = factor.solve_lu_device(f, x)
        t = timed(lambda: factor.solve_lu_device(f, x))
        print(f"{cfg} systems={A.nsys} n={A.n} {'csc' if csc else 'rows'}: {t:8.3f} ms "
              f"{byt / t / 1e6:8.1f} GB/s  ({1e6 * t / (2 * A.n):.1f} ns/column)", flush=True)
    same = torch.equal(out[True].view(torch.int64), out[False].view(torch.int64))
    print("  bit-identical" if same else "  MISMATCH")


if __name__ == "__main__":
    if len(sys.argv) > 1:
        main(sys.argv[1])
        raise SystemExit
    main("c1")
    main("c2")
    main("c4", 1)
    main("c4", 512)
