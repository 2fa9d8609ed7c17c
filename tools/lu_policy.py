"""Complete LU of c4 batches: frontal kernel vs compact column pipeline, by batch size."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1504_06768_b200 import _lib, configs, factor, liouville, ordering  # noqa: E402


def main(counts="1,16,64,148,200,256,296,370,444,512", reps=5):
    for count in [int(x) for x in counts.split(",")]:
        L = liouville.build_liouvillian_batch([configs.jc_sweep(i) for i in range(count)])
        sh = liouville.shift(L)
        fwd, inv = ordering.rcm_device(sh.matrix)
        A = ordering.permute(sh.matrix, fwd, inv)
        row = []
        for name, env in (("frontal", {"RHOSOLVE_FRONTAL": "1", "RHOSOLVE_COMPACT": "0"}),
                          ("compact", {"RHOSOLVE_FRONTAL": "0", "RHOSOLVE_COMPACT": "1"}),
                          ("general", {"RHOSOLVE_FRONTAL": "0", "RHOSOLVE_COMPACT": "0"})):
            os.environ.update(env)
            ts = []
            for _ in range(int(reps)):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                factor.factor_batch(A, 0.0, float("inf"))
                torch.cuda.synchronize()
                ts.append(time.perf_counter() - t0)
            ts.sort()
            row.append(f"{name} {1e3 * ts[len(ts) // 2]:.2f} (min {1e3 * ts[0]:.2f}, max {1e3 * ts[-1]:.2f})")
        print(f"systems {count:4d}: " + " | ".join(row), flush=True)


if __name__ == "__main__":
    main(*sys.argv[1:])
