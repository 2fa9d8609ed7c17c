"""Per-column phase clocks of system 0 while the whole c4 batch (512 complete
LUs) factors -- where the batch factorization's time goes (tuning)."""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1504_06768_b200 import _lib, configs, factor, liouville, ordering  # noqa: E402


def main(count="512"):
    count = int(count)
    L = liouville.build_liouvillian_batch([configs.jc_sweep(i) for i in range(count)])
    sh = liouville.shift(L)
    fwd, inv = ordering.rcm_device(sh.matrix)
    A = ordering.permute(sh.matrix, fwd, inv)
    n = A.n
    lib = _lib.load()
    lib.rs_debug_factor_probe.argtypes = [ctypes.c_void_p]
    buf = torch.zeros(n * 6, dtype=torch.int64, device="cuda")
    factor.factor_batch(A, 0.0, float("inf"))
    lib.rs_debug_factor_probe(ctypes.c_void_p(buf.data_ptr()))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    factor.factor_batch(A, 0.0, float("inf"))
    e1.record()
    torch.cuda.synchronize()
    lib.rs_debug_factor_probe(None)
    print(f"systems {count}: factor_batch {e0.elapsed_time(e1):.2f} ms")
    p = buf.view(n, 6).cpu().numpy().astype(np.int64)
    fin = p[:, 4]
    gap = np.diff(fin)
    print("system 0 span cycles", fin[-1] - p[0, 0], "per column median/mean", np.median(gap),
          gap.mean(), "p90", np.percentile(gap, 90))
    ready = p[1:, 1] - fin[:-1]
    print("median: ready-after-prev", np.median(ready), "pivot", np.median(p[:, 2] - p[:, 1]),
          "cap", np.median(p[:, 3] - p[:, 2]), "emit", np.median(p[:, 4] - p[:, 3]))
    print("mean:   ready-after-prev", ready.mean(), "pivot", (p[:, 2] - p[:, 1]).mean(),
          "emit", (p[:, 4] - p[:, 3]).mean(), "work start->ready", (p[:, 1] - p[:, 0]).mean())
    print("fraction of columns ready only after the previous column published",
          (ready > 0).mean())


if __name__ == "__main__":
    main(*sys.argv[1:])
