"""SpMV bandwidth on the c4 batch (158 MB) and a 4x replicated batch
(~630 MB, beyond L2), event-timed with the L2 flushed (tuning)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1504_06768_b200 import _lib, configs, liouville, ordering  # noqa: E402
from paper_1504_06768_b200.sparse import DeviceCSR  # noqa: E402


def timed(fn, reps=10):
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
    ts.sort()
    return ts[len(ts) // 2]


def run(A, label):
    x = torch.randn(A.n * A.nsys, dtype=torch.complex128, device="cuda")
    y = torch.empty_like(x)
    f = lambda: _lib.call("rs_csr_matvec", A.nsys, A.n, _lib.ptr(A.row_ptr), _lib.ptr(A.col_idx),  # noqa: E731
                          _lib.ptr(A.values), _lib.ptr(x), _lib.ptr(y), _lib.stream_ptr())
    t = timed(f)
    byt = 20 * A.nnz + 4 * (A.n * A.nsys + 1) + 32 * A.n * A.nsys
    print(f"{label}: nnz={A.nnz} {byt / 1e6:.1f} MB  {t * 1e3:.1f} us  {byt / t / 1e6:.0f} GB/s",
          flush=True)


def main():
    L = liouville.build_liouvillian_batch([configs.jc_sweep(i) for i in range(512)])
    sh = liouville.shift(L)
    fwd, inv = ordering.rcm_device(sh.matrix)
    A = ordering.permute(sh.matrix, fwd, inv)
    run(A, "c4 batch x512")
    R = 4
    nnz = A.nnz
    rp = torch.cat([A.row_ptr[:-1] + r * nnz for r in range(R)] +
                   [torch.tensor([R * nnz], dtype=torch.int32, device="cuda")])
    B = DeviceCSR(A.n, A.nsys * R, rp, A.col_idx.repeat(R), A.values.repeat(R))
    run(B, "c4 batch x2048")
    M = liouville.build_modified(L)
    run(M.matrix, "c4 modified x512 (trace rows)")


if __name__ == "__main__":
    main()
