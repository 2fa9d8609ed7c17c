"""Wall time of the c4 batch complete-LU factorization (512 systems), frontal
kernel vs the column pipeline (RHOSOLVE_FRONTAL=0)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1504_06768_b200 import _lib, configs, factor, liouville, ordering  # noqa: E402


def main(count=512, reps=5, modes="101"):
    L = liouville.build_liouvillian_batch([configs.jc_sweep(i) for i in range(int(count))])
    sh = liouville.shift(L)
    fwd, inv = ordering.rcm_device(sh.matrix)
    A = ordering.permute(sh.matrix, fwd, inv)
    for mode in modes:
        os.environ["RHOSOLVE_FRONTAL"] = mode
        ts = []
        for _ in range(int(reps)):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            f = factor.factor_batch(A, 0.0, float("inf"))
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        import ctypes
        ph = (ctypes.c_double * 4)()
        lib = _lib.load()
        lib.rs_debug_frontal_probe(1, None)
        factor.factor_batch(A, 0.0, float("inf"))
        torch.cuda.synchronize()
        lib.rs_debug_frontal_probe(0, ph)
        print("cycles/step P1 P2 P3:", [round(x) for x in ph[:3]])
        print(f"frontal={mode} taken={_lib.load().rs_debug_frontal_taken()} "
              f"median {1e3 * sorted(ts)[len(ts) // 2]:.2f} ms  min {1e3 * min(ts):.2f} ms "
              f"fill {f.fill_factors[:2]}  all ms {[round(1e3 * t, 1) for t in ts]}")


if __name__ == "__main__":
    main(*sys.argv[1:])
