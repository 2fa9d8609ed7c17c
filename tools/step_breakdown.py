"""Where a c4 bench step spends its time: every C-ABI call is timed with a
device synchronisation after it (host launch + device time), torch work and
Python bookkeeping are what remains of each stage."""
import collections
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1504_06768_b200 import _lib, configs, liouville, steady  # noqa: E402


def main(count=512, reps=3, sync_calls=1):
    count, reps, sync_calls = int(count), int(reps), int(sync_calls)
    L = liouville.build_liouvillian_batch([configs.jc_sweep(i) for i in range(count)])
    seeds = [2 + i for i in range(count)]
    kw = dict(tol=1e-12, inner="direct", ordering_name="rcm")
    for _ in range(2):
        steady.inverse_power_batch(L, seeds, **kw)
    acc = collections.OrderedDict()
    orig = _lib.call

    def timed_call(name, *a):
        if sync_calls:
            torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = orig(name, *a)
        if sync_calls:
            torch.cuda.synchronize()
        acc[name] = acc.get(name, 0.0) + time.perf_counter() - t0
        acc[name + "#"] = acc.get(name + "#", 0) + 1
        return r

    _lib.call = timed_call
    for mod in (steady, liouville):
        pass
    import paper_1504_06768_b200.factor as F
    import paper_1504_06768_b200.ordering as Od
    import paper_1504_06768_b200.sparse as Sp
    tot = 0.0
    stages = [0.0, 0.0, 0.0]
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = steady.inverse_power_batch(L, seeds, **kw)
        torch.cuda.synchronize()
        tot += time.perf_counter() - t0
        stages[0] += res[0].build_time
        stages[1] += res[0].factor_time
        stages[2] += res[0].solve_time
    _lib.call = orig
    print(f"step {1e3 * tot / reps:.2f} ms (sync after every C call: {bool(sync_calls)}); stages "
          f"build {1e3 * stages[0] / reps:.2f} factor {1e3 * stages[1] / reps:.2f} "
          f"solve {1e3 * stages[2] / reps:.2f}")
    s = 0.0
    for k, v in acc.items():
        if k.endswith("#"):
            continue
        s += v
        print(f"  {k:28s} x{acc[k + '#'] // reps:3d} {1e3 * v / reps:8.3f} ms")
    print(f"  C-ABI calls total {1e3 * s / reps:.2f} ms; torch + Python {1e3 * (tot - s) / reps:.2f} ms")


if __name__ == "__main__":
    main(*sys.argv[1:])
