"""Per-column phase timing of the pipelined ILUTP kernel (tuning experiment).
Phases (clock64 on the CTA's SM): 0 start of column, 1 frontier reached k
(all updates applied), 2 pivot chosen, 3 drop/cap done, 4 published."""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1504_06768_b200 import _lib, configs, factor, liouville, ordering  # noqa: E402


def main(cfg="c2"):
    c = configs.CONFIGS[cfg]
    H, cops = c["build"]()
    L = liouville.build_liouvillian(H, cops)
    sh = liouville.shift(L)
    fwd, inv = ordering.rcm_device(sh.matrix)
    A = ordering.permute(sh.matrix, fwd, inv)
    n = A.n
    lib = _lib.load()
    buf = torch.zeros(n * 6, dtype=torch.int64, device="cuda")
    lib.rs_debug_factor_probe.argtypes = [ctypes.c_void_p]
    factor.factor_batch(A, c["d"], c["p"])  # warm
    lib.rs_debug_factor_probe(ctypes.c_void_p(buf.data_ptr()))
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    factor.factor_batch(A, c["d"], c["p"])
    t1.record()
    torch.cuda.synchronize()
    lib.rs_debug_factor_probe(None)
    print("factor_batch ms", t0.elapsed_time(t1))
    p = buf.view(n, 6).cpu().numpy().astype(np.int64)
    fin = p[:, 4]
    gap = np.diff(fin)  # cycles between consecutive column completions
    ready_after_prev = p[1:, 1] - fin[:-1]  # column k frontier reached after k-1 published
    print("cycles per column (median/mean):", np.median(gap), gap.mean())
    print("tail phases median: ready-after-prev", np.median(ready_after_prev),
          "pivot", np.median(p[:, 2] - p[:, 1]), "drop", np.median(p[:, 3] - p[:, 2]),
          "emit", np.median(p[:, 4] - p[:, 3]))
    late = p[1:, 1] > fin[:-1]
    print("fraction of columns whose updates finish after the previous column:", late.mean())
    print("median column work (start->ready):", np.median(p[:, 1] - p[:, 0]))




def distribution(cfg="c2"):
    """Percentiles of per-column critical-path cycles and the phase split of
    the slowest decile."""
    import ctypes
    c = configs.CONFIGS[cfg]
    L = liouville.build_liouvillian(*c["build"]())
    sh = liouville.shift(L)
    fwd, inv = ordering.rcm_device(sh.matrix)
    A = ordering.permute(sh.matrix, fwd, inv)
    n = A.n
    lib = _lib.load()
    buf = torch.zeros(n * 6, dtype=torch.int64, device="cuda")
    lib.rs_debug_factor_probe.argtypes = [ctypes.c_void_p]
    factor.factor_batch(A, c["d"], c["p"])
    lib.rs_debug_factor_probe(ctypes.c_void_p(buf.data_ptr()))
    f = factor.factor_batch(A, c["d"], c["p"])
    torch.cuda.synchronize()
    lib.rs_debug_factor_probe(None)
    p = buf.view(n, 6).cpu().numpy().astype(np.int64)
    gap = np.diff(p[:, 4])
    print("per-column cycles percentiles 10/50/90/99:", np.percentile(gap, [10, 50, 90, 99]))
    slow = np.argsort(gap)[-len(gap) // 10:] + 1
    ready = p[slow, 1] - p[slow - 1, 4]
    print("slowest decile: mean gap", gap[slow - 1].mean(), "ready-after-prev", ready.mean(),
          "pivot", (p[slow, 2] - p[slow, 1]).mean(), "emit", (p[slow, 4] - p[slow, 3]).mean(),
          "share of total", gap[slow - 1].sum() / gap.sum())
    lp = f.raw[0][:n + 1].cpu().numpy()
    up = f.raw[3][:n + 1].cpu().numpy()
    lcol, ucol = np.diff(lp), np.diff(up)
    print("L/U column sizes slow decile", lcol[slow].mean(), ucol[slow].mean(), "overall",
          lcol.mean(), ucol.mean())


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "dist":
        distribution(*sys.argv[2:])
    else:
        main(*sys.argv[1:])
