"""Config 5 (two coupled Kerr cavities) through the sharded large-system path.
    python tools/run_c5.py [N=40] [blocks=8] [max_iter=1000] [d=1e-5] [p=10]
Prints per-stage times, iteration counts and the plain-L residual."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1504_06768_b200 import configs, liouville, sharded  # noqa: E402


def main(N="40", blocks="8", max_iter="1000", d="1e-5", p="10"):
    N, blocks, max_iter, d, p = int(N), int(blocks), int(max_iter), float(d), float(p)
    t = time.perf_counter()
    H, c = configs.kerr_kerr(N=N)
    t_ops = time.perf_counter() - t
    torch.cuda.synchronize()
    t = time.perf_counter()
    L = liouville.build_liouvillian(H, c)
    torch.cuda.synchronize()
    t_asm = time.perf_counter() - t
    print(f"N={N} n={L.n} nnz={L.matrix.nnz} host ops {t_ops:.2f}s assembly {t_asm:.3f}s",
          flush=True)
    res = sharded.inverse_power_sharded(L, tol=1e-10, d=d, p=p, seed=3, blocks=blocks,
                                        max_iter=max_iter, log=lambda m: print(m, flush=True))
    print(f"build(shift+rcm+permute+shard) {res.build_time:.2f}s factor {res.factor_time:.2f}s "
          f"solve {res.solve_time:.2f}s outer {res.iterations} inner {res.inner_iterations} "
          f"residual {res.residual:.3e} extra {res.extra}", flush=True)


if __name__ == "__main__":
    main(*sys.argv[1:])
