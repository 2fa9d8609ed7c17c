"""Time the SELL lane-per-row triangular sweep against the warp-per-row sweep
on one system's factors (single CTA), checking both give identical bits."""
import ctypes
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1504_06768_b200 import _lib, configs, factor, liouville, ordering  # noqa: E402


def sell(n, rp, ci, v, upper):
    nsl = (n + 31) // 32
    sptr = torch.empty(nsl + 1, dtype=torch.int32, device="cuda")
    tot = ctypes.c_int64(0)
    st = _lib.stream_ptr()
    _lib.call("rs_sell_build", 1, n, upper, _lib.ptr(rp), _lib.ptr(ci), _lib.ptr(v),
              _lib.ptr(sptr), None, None, ctypes.byref(tot), st)
    sci = torch.empty(tot.value, dtype=torch.int32, device="cuda")
    sv = torch.empty(tot.value, dtype=torch.complex128, device="cuda")
    _lib.call("rs_sell_build", 1, n, upper, _lib.ptr(rp), _lib.ptr(ci), _lib.ptr(v),
              _lib.ptr(sptr), _lib.ptr(sci), _lib.ptr(sv), ctypes.byref(tot), st)
    return sptr, sci, sv, tot.value


def main(cfg="c2"):
    if cfg == "c4":
        H, cops = configs.jc_sweep(0)
        d, p = 0.0, math.inf
    else:
        c = configs.CONFIGS[cfg]
        H, cops = c["build"]()
        d, p = c["d"], c["p"]
    L = liouville.build_liouvillian(H, cops)
    sh = liouville.shift(L)
    fwd, inv = ordering.rcm_device(sh.matrix)
    A = ordering.permute(sh.matrix, fwd, inv)
    f = factor.factor_batch(A, d, p).ensure_rows()
    lib = _lib.load()
    fn = lib.rs_debug_tri_probe
    fn.argtypes = [ctypes.c_int] + [ctypes.c_void_p] * 6 + [ctypes.c_int] * 4 + [ctypes.c_void_p]
    n = A.n
    x = torch.randn(n, dtype=torch.complex128, device="cuda")
    out = torch.empty_like(x)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream()
    smem_ok = 16 * n <= 200 * 1024
    for which, (rp, ci, v) in ((0, (f.L_rp, f.L_ci, f.L_v)), (1, (f.U_rp, f.U_ci, f.U_v))):
        nnz = int(rp[-1].item())
        sp, sci, sv, tot = sell(n, rp, ci, v, which)
        print(f"{cfg} {'LU'[which]}: n={n} nnz={nnz} sell padded={tot} ({tot / max(nnz, 1):.3f}x)")
        ref = None
        lib.rs_debug_tri_backoff.argtypes = [ctypes.c_uint, ctypes.c_uint]
        for variant, threads, nap in ((1, 512, (0, 0)), (1, 512, (20, 200)), (1, 512, (50, 500)),
                                      (1, 512, (100, 1000)), (1, 512, (20, 2000)),
                                      (1, 256, (0, 0)), (1, 256, (20, 200)), (1, 1024, (50, 500))):
            lib.rs_debug_tri_backoff(*nap)
            args = (sp, sci, sv) if variant >= 3 else (rp, ci, v)
            ts = []
            for rep in range(4):
                flush.zero_()
                torch.cuda.synchronize()
                torch.cuda._sleep(50_000)
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(st)
                rc = fn(n, args[0].data_ptr(), args[1].data_ptr(), args[2].data_ptr(),
                        f.rdiag.data_ptr(), x.data_ptr(), out.data_ptr(), which, variant,
                        1 if smem_ok else 0, threads, ctypes.c_void_p(st.cuda_stream))
                b.record(st)
                torch.cuda.synchronize()
                assert rc == 0, _lib.load().rs_last_error()
                ts.append(a.elapsed_time(b))
            o = out.clone()
            same = "" if ref is None else ("bit-identical" if torch.equal(o.view(torch.int64), ref.view(torch.int64)) else "MISMATCH")
            if ref is None:
                ref = o
            t = min(ts[1:])
            print(f"  variant={variant} nap={nap} threads={threads:4d} {t:8.3f} ms {1e6 * t / n:7.1f} ns/row "
                  f"{20 * nnz / t / 1e6:8.1f} GB/s {same}", flush=True)


if __name__ == "__main__":
    for c in (sys.argv[1:] or ["c2"]):
        main(c)
