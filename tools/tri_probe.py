"""Time lower / upper triangular sweeps of the c2 preconditioner in isolation
for each row-mapping variant (tuning experiment)."""
import ctypes
import os
import sys

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
    f = factor.factor_batch(A, c["d"], c["p"])
    lib = _lib.load()
    fn = lib.rs_debug_tri_probe
    fn.argtypes = [ctypes.c_int] + [ctypes.c_void_p] * 6 + [ctypes.c_int] * 4 + [ctypes.c_void_p]
    n = A.n
    x = torch.randn(n, dtype=torch.complex128, device="cuda")
    out = torch.empty_like(x)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream()
    lib.rs_debug_tri_backoff.argtypes = [ctypes.c_uint, ctypes.c_uint]
    for which, (rp, ci, v) in ((0, (f.L_rp, f.L_ci, f.L_v)), (1, (f.U_rp, f.U_ci, f.U_v))):
      for nmin, nmax in ((0, 0),):
        lib.rs_debug_tri_backoff(nmin, nmax)
        for variant in (1, 2):
            for smem_buf in (1,):
                for threads in (256, 512, 1024):
                    for hot in (0,):
                        ts = []
                        for rep in range(4):
                            if not hot:
                                flush.zero_()
                            a = torch.cuda.Event(enable_timing=True)
                            b = torch.cuda.Event(enable_timing=True)
                            torch.cuda.synchronize()
                            a.record(st)
                            rc = fn(n, rp.data_ptr(), ci.data_ptr(), v.data_ptr(),
                                    f.rdiag.data_ptr(), x.data_ptr(), out.data_ptr(), which,
                                    variant, smem_buf, threads, ctypes.c_void_p(st.cuda_stream))
                            b.record(st)
                            torch.cuda.synchronize()
                            assert rc == 0
                            ts.append(a.elapsed_time(b))
                        print(f"nap={nmin}/{nmax} {'LU'[which]} variant={'thread' if variant == 0 else 'warp  '} "
                              f"smem={smem_buf} threads={threads:4d} l2={'hot ' if hot else 'cold'}"
                              f" {min(ts[1:]):8.3f} ms  ({1e6 * min(ts[1:]) / n:7.1f} ns/row)",
                              flush=True)


if __name__ == "__main__":
    main(*sys.argv[1:])
