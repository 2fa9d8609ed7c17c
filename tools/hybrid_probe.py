"""c4 batch complete LU: frontal + pipeline sharing the SMs (RHOSOLVE_HYBRID_F
leading systems frontal, the rest pipeline CTAs beside the fronts), timing and
bit equality with the pure column pipeline."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1504_06768_b200 import _lib, configs, factor, liouville, ordering  # noqa: E402


def snapshot(f):
    """valid part of every raw array (entries beyond a column pointer's end are scratch)"""
    Lp, Li, Lx, Up, Ui, Ux = f.raw
    n, B = f.n, f.nsys
    lp = Lp.view(B, n + 1).cpu()
    up = Up.view(B, n + 1).cpu()
    out = [lp, up, f.pinv.cpu()]
    li, lx = Li.view(B, -1).cpu(), Lx.view(B, -1).cpu()
    ui, ux = Ui.view(B, -1).cpu(), Ux.view(B, -1).cpu()
    for b in range(0, B, max(1, B // 64)):
        out += [li[b, :lp[b, n]].clone(), torch.view_as_real(lx[b, :lp[b, n]]).view(torch.int64).clone(),
                ui[b, :up[b, n]].clone(), torch.view_as_real(ux[b, :up[b, n]]).view(torch.int64).clone()]
    return out


def compact(count=512, reps=7, capx=""):
    """RHOSOLVE_COMPACT=1 (compact shared-memory kernel) against the general pipeline."""
    count, reps = int(count), int(reps)
    L = liouville.build_liouvillian_batch([configs.jc_sweep(i) for i in range(count)])
    sh = liouville.shift(L)
    fwd, inv = ordering.rcm_device(sh.matrix)
    A = ordering.permute(sh.matrix, fwd, inv)
    os.environ["RHOSOLVE_FRONTAL"] = "0"
    os.environ["RHOSOLVE_COMPACT"] = "0"
    ref = snapshot(factor.factor_batch(A, 0.0, float("inf")))
    for mode in ("0", "1"):
        os.environ["RHOSOLVE_COMPACT"] = mode
        if capx and mode == "1":
            os.environ["RHOSOLVE_COMPACT_CAPX"] = capx
        ts = []
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            f = factor.factor_batch(A, 0.0, float("inf"))
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        got = snapshot(f)
        same = all(torch.equal(a, b) for a, b in zip(ref, got))
        print(f"compact={mode} systems {count} median {1e3 * sorted(ts)[len(ts) // 2]:.2f} ms "
              f"min {1e3 * min(ts):.2f} ms bit-equal {same} ok {bool(f.ok.all()) if hasattr(f.ok, 'all') else f.ok} "
              f"all {[round(1e3 * t, 1) for t in ts]}", flush=True)


def main(count=512, reps=7, fs="0,148,222,296,330,370"):
    if fs == "compact" or str(fs).startswith("compact"):
        return compact(count, reps, str(fs)[8:])
    count, reps = int(count), int(reps)
    L = liouville.build_liouvillian_batch([configs.jc_sweep(i) for i in range(count)])
    sh = liouville.shift(L)
    fwd, inv = ordering.rcm_device(sh.matrix)
    A = ordering.permute(sh.matrix, fwd, inv)
    os.environ["RHOSOLVE_FRONTAL"] = "0"
    os.environ["RHOSOLVE_HYBRID_F"] = "0"
    ref = snapshot(factor.factor_batch(A, 0.0, float("inf")))
    os.environ.pop("RHOSOLVE_FRONTAL")
    for F in [int(x) for x in fs.split(",")]:
        os.environ["RHOSOLVE_HYBRID_F"] = str(F)
        ts = []
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            f = factor.factor_batch(A, 0.0, float("inf"))
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        got = snapshot(f)
        same = all(torch.equal(a, b) for a, b in zip(ref, got))
        print(f"F={F:4d} taken={_lib.load().rs_debug_frontal_taken():4d} median "
              f"{1e3 * sorted(ts)[len(ts) // 2]:.2f} ms min {1e3 * min(ts):.2f} ms bit-equal {same} "
              f"all {[round(1e3 * t, 1) for t in ts]}", flush=True)


if __name__ == "__main__":
    main(*sys.argv[1:])
