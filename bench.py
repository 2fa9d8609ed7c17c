#!/usr/bin/env python
"""Benchmark: steady-state solves/sec of the doubly-iterative inverse-power
method (BASELINE.json metric) on B200, plus SpMV / ILU-apply HBM GB/s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c1|c4]
    python bench.py --impl reference ...      # the reference CPU path

A step is one full `inverse_power(L, inner="iterative", solver="bicgstab",
ordering_name="rcm", ...)` call from an assembled Liouvillian to rho
(shift, RCM, permute, ILUTP, the device-resident inner/outer iteration,
unpermute + post-processing).  Default workload = BASELINE configs[1] (c2,
driven JC N=40 x qubit, n = 6400).  c1..c3 do not shard: N GPUs run N
independent replicas (scaling "weak").  Rank 0 prints one JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (config key, builder kwargs, solve kwargs, D)
    "c2": ("c2", {}, dict(tol=1e-12, inner="iterative", ordering_name="rcm",
                          solver="bicgstab", d=1e-4, p=300.0, seed=1), 80),
    "c1": ("c1", {}, dict(tol=1e-12, inner="iterative", ordering_name="rcm",
                          solver="bicgstab", d=1e-5, p=10.0, seed=0), 20),
    "c4": ("c4", {}, dict(tol=1e-12, inner="direct", ordering_name="rcm"), 40),
}
DESCR = {
    "c2": "c2: driven Jaynes-Cummings N=40 x qubit (n=6400), inverse_power inner=BiCGStab, "
          "ILUTP(d=1e-4,p=300) under RCM, tol=1e-12, seed=1",
    "c1": "c1: driven Kerr N=20 (n=400), inverse_power inner=BiCGStab, ILUTP(1e-5,10), RCM, "
          "tol=1e-12, seed=0",
    "c4": "c4: 512-instance JC sweep N=20 x qubit (n=1600 each), inverse_power inner=direct "
          "(complete LU), RCM, tol=1e-12, seeds 2+i",
}


def build_inputs(cfg):
    from paper_1504_06768_b200 import configs
    key, bkw, _, _ = WORKLOADS[cfg]
    if cfg == "c4":
        return [configs.jc_sweep(i) for i in range(512)]
    return [configs.CONFIGS[key]["build"](**bkw)]


# ------------------------------------------------------------ reference ----
def _ref_path():
    p = os.path.join(ROOT, "oracle", "_ref")
    return p if os.path.isdir(os.path.join(p, "rhosolve")) else None


def _ref_worker(args):
    cfg, count = args
    os.environ["OMP_NUM_THREADS"] = "1"
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    rp = _ref_path()
    if rp and rp not in sys.path:
        sys.path.insert(0, rp)
    from rhosolve import liouville as RL, operators as RO, steady as RSt
    from paper_1504_06768_b200 import configs
    _, bkw, skw, _ = WORKLOADS[cfg]
    if cfg == "c4":
        models = [configs.jc_sweep(i % 512, ops=RO) for i in range(count)]
    else:
        models = [configs.CONFIGS[WORKLOADS[cfg][0]]["build"](**bkw, ops=RO)] * count
    Ls = [RL.build_liouvillian(H, c) for H, c in models]
    t = time.perf_counter()
    for k, L in enumerate(Ls):
        kw = dict(skw)
        if cfg == "c4":
            kw["seed"] = 2 + (k % 512)
        RSt.inverse_power(L, **kw)
    return time.perf_counter() - t


def _oracle_worker(args):
    cfg, count = args
    from oracle import oracle as O
    from paper_1504_06768_b200 import configs
    _, bkw, skw, D = WORKLOADS[cfg]
    H, c = (configs.jc_sweep(0) if cfg == "c4"
            else configs.CONFIGS[WORKLOADS[cfg][0]]["build"](**bkw))
    L = O.build_liouvillian(H.matrix, [x.matrix for x in c])
    kw = {k: v for k, v in skw.items() if k != "ordering_name"}
    t = time.perf_counter()
    for _ in range(count):
        O.inverse_power(L, D, **kw)
    return time.perf_counter() - t


def cpu_solves_per_sec(cfg, workers, target_s):
    """Time the reference (oracle/_ref) -- or the oracle port when the
    reference build is absent -- for about target_s seconds per worker."""
    kind = "reference" if _ref_path() else "port"
    fn = _ref_worker if kind == "reference" else _oracle_worker
    probe = fn((cfg, 1))
    count = max(1, int(target_s / max(probe, 1e-3)))
    if workers == 1:
        dt = fn((cfg, count))
        return count / dt, kind, count, probe
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    with ctx.Pool(workers) as pool:
        t = time.perf_counter()
        pool.map(fn, [(cfg, count)] * workers)
        wall = time.perf_counter() - t
    return workers * count / wall, kind, count, probe


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg = args.config
    workers = os.cpu_count() or 1
    per_step = []
    kind = "reference" if _ref_path() else "port"
    fn = _ref_worker if kind == "reference" else _oracle_worker
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    with ctx.Pool(workers) as pool:
        for s in range(args.warmup + args.steps):
            t = time.perf_counter()
            pool.map(fn, [(cfg, 1)] * workers)
            dt = time.perf_counter() - t
            if s >= args.warmup:
                per_step.append(dt)
    total = sum(per_step)
    value = workers * len(per_step) / total
    line = {
        "impl": "reference", "metric": "steady-state solves/sec", "value": value,
        "unit": "solves/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / len(per_step), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": {"workload": DESCR[cfg], "parallelism": f"{workers} CPU processes"},
        "cpu_baseline": {"value": value, "unit": "solves/s", "cores": workers, "kind": kind,
                         "sample": f"{args.steps} steps x {workers} processes x 1 solve "
                                   "(OMP/OpenBLAS threads = 1 per process)"},
        "e2e": {"value": value, "unit": "solves/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU ----
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peak():
    for p in (os.path.join(ROOT, "MEASURED_PEAKS.json"),):
        try:
            with open(p) as fh:
                return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
        except (OSError, KeyError, ValueError):
            pass
    return 6650.0, "fallback (B200_PROFILING.md)"


def kernel_timings(L, skw, torch, lib_mod):
    """Event-timed standalone launches on the c2 matrices: the ILUTP kernel,
    the fused solver kernel, SpMV and ILU apply (each on the launching
    stream, warm, with an L2 flush before every timed launch)."""
    from paper_1504_06768_b200 import factor, liouville, ordering, steady
    from paper_1504_06768_b200 import _lib
    st = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def timed(fn, reps=5):
        ts = []
        for _ in range(reps):
            flush.zero_()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record(st)
            fn()
            b.record(st)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e-3)
        return statistics.median(ts)

    sh = liouville.shift(L)
    fwd, inv = ordering.rcm_device(sh.matrix)
    A = ordering.permute(sh.matrix, fwd, inv)
    P = ordering.permute(L.matrix, fwd, inv)
    n, nnz = A.n, A.nnz
    out = {}
    # ILUTP: the rs_factorize launch alone
    Ap, Ai, Ax = factor._transpose(A)
    rn = torch.empty(n, dtype=torch.float64, device="cuda")
    _lib.call("rs_row_norms", 1, n, _lib.ptr(A.row_ptr), _lib.ptr(A.values), _lib.ptr(rn),
              _lib.stream_ptr())
    f = factor.factor_batch(A, skw.get("d", 0.0), skw.get("p", float("inf")))
    capL, capU = f.capL, f.capU
    import math
    cap = int(math.ceil(skw["p"] * nnz / n)) if "p" in skw else -1
    Lp = torch.zeros(n + 1, dtype=torch.int32, device="cuda")
    Up = torch.zeros_like(Lp)
    Li = torch.empty(capL, dtype=torch.int32, device="cuda")
    Lx = torch.empty(capL, dtype=torch.complex128, device="cuda")
    Ui = torch.empty(capU, dtype=torch.int32, device="cuda")
    Ux = torch.empty(capU, dtype=torch.complex128, device="cuda")
    pinv = torch.empty(n, dtype=torch.int32, device="cuda")
    state = torch.zeros(3, dtype=torch.int32, device="cuda")

    def run_fact():
        state.zero_()
        _lib.call("rs_factorize", 1, n, _lib.ptr(Ap), _lib.ptr(Ai), _lib.ptr(Ax), None,
                  float(skw.get("d", 0.0)), cap, _lib.ptr(rn), _lib.ptr(Lp), _lib.ptr(Li),
                  _lib.ptr(Lx), capL, _lib.ptr(Up), _lib.ptr(Ui), _lib.ptr(Ux), capU,
                  _lib.ptr(pinv), _lib.ptr(state), _lib.stream_ptr())

    t_fact = timed(run_fact, reps=3)
    lnnz, unnz = int(f.lnnz[0]), int(f.unnz[0])
    out["ilutp"] = {"seconds": t_fact, "bytes": 20 * nnz + 20 * (lnnz + unnz) + 8 * (n + 1),
                    "note": "one warp per system, column-sequential left-looking ILUTP"}
    # SpMV
    x = torch.randn(n, dtype=torch.complex128, device="cuda")
    y = torch.empty_like(x)

    def run_spmv():
        _lib.call("rs_csr_matvec", 1, n, _lib.ptr(A.row_ptr), _lib.ptr(A.col_idx),
                  _lib.ptr(A.values), _lib.ptr(x), _lib.ptr(y), _lib.stream_ptr())

    b_spmv = 20 * nnz + 4 * (n + 1) + 32 * n
    out["spmv"] = {"seconds": timed(run_spmv, reps=20), "bytes": b_spmv}
    # ILU apply
    nLU = int(f.L_ci.numel()) + int(f.U_ci.numel())

    def run_apply():
        factor.solve_lu_device(f, x)

    b_apply = 20 * (lnnz + unnz) + 72 * n
    out["ilu_apply"] = {"seconds": timed(run_apply, reps=10), "bytes": b_apply,
                        "nnz_offdiag": nLU}
    # fused solver kernel (whole inner/outer iteration, one launch)
    x0 = torch.from_numpy(steady.start_vector(n, skw.get("seed", 0))).cuda()
    mode = _lib.INV_BICGSTAB if skw.get("solver") == "bicgstab" else _lib.INV_GMRES
    res = {}

    def run_solver():
        xs, stt = steady._solve(mode, A, P, f, x0, skw["tol"], 1000, 20, True)
        res["st"] = stt

    t_solver = timed(run_solver, reps=3)
    s = res["st"][0]
    its = int(s["inner_total"])
    outer = int(s["outer"])
    # per inner BiCGStab iteration: 2 SpMV + 2 applies + ~13 vector passes
    # (fused), plus per outer step psolve(b) + 2 residual SpMVs.
    b_solver = (its * (2 * b_spmv + 2 * b_apply + 16 * n * 13)
                + outer * (b_apply + 2 * b_spmv) + b_apply)
    out["solver"] = {"seconds": t_solver, "bytes": b_solver, "inner_iterations": its,
                     "outer": outer}
    return out


def run_gpu(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    from paper_1504_06768_b200 import _lib, liouville, steady
    from paper_1504_06768_b200.sparse import from_host
    lib = _lib.load()
    lib.rs_launch_count.restype = __import__("ctypes").c_longlong

    cfg = args.config
    _, _, skw, D = WORKLOADS[cfg]
    models = build_inputs(cfg)
    if cfg == "c4":
        L = liouville.build_liouvillian_batch(models)
        seeds = [2 + i for i in range(len(models))]

        def step(Lx):
            return steady.inverse_power_batch(Lx, seeds, **skw)
        per_step_solves = len(models)
    else:
        L = liouville.build_liouvillian(*models[0])

        def step(Lx):
            return [steady.inverse_power(Lx, **skw)]
        per_step_solves = 1
    host_L = [L.matrix.system(b) for b in range(L.nsys)]

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream()
    for _ in range(args.warmup):
        step(L)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    times = []
    last = None
    l0 = lib.rs_launch_count()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record(st)
            last = step(L)
            b.record(st)
            torch.cuda.synchronize()
            times.append(a.elapsed_time(b) * 1e-3)
    launches = (lib.rs_launch_count() - l0) // max(args.steps, 1)
    total = sum(times)
    if dist:
        t = torch.tensor([total], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total = float(t.item())
        dist.barrier()
    value = world * per_step_solves * args.steps / total

    # e2e: public API from HOST buffers (pinned) -> rho on the host, per step
    e2e_times, h2d, d2h = [], 0, 0
    pinned = []
    for m in host_L:
        pinned.append(m)
    for s in range(max(2, min(args.steps, 5))):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        Lh = from_host(pinned)
        Ls = liouville.LiouvillianSystem(Lh, D, "plain")
        res = step(Ls)
        torch.cuda.synchronize()
        e2e_times.append(time.perf_counter() - t0)
        h2d = sum(4 * (m.nrows + 1) + 20 * m.nnz for m in host_L) + 16 * sum(m.nrows for m in host_L)
        d2h = sum(16 * D * D + 40 for _ in res)
    e2e_value = world * per_step_solves / statistics.median(e2e_times)

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return 0

    # roofline: dominant kernel of a step, timed standalone
    peak, peak_src = measured_peak()
    kt = {}
    if cfg != "c4":
        kt = kernel_timings(L, skw, torch, lib)
    kernels = {}
    for k, v in kt.items():
        gbs = v["bytes"] / v["seconds"] / 1e9
        kernels[k] = dict(v, achieved_gbs=gbs, frac=gbs / peak)
    dom = max(kt, key=lambda k: kt[k]["seconds"]) if kt else None
    roof = None
    if dom:
        ach = kernels[dom]["achieved_gbs"]
        roof = {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": peak, "unit": "GB/s",
                "frac": ach / peak, "traffic": None, "peak_source": peak_src,
                "share_of_step": kt[dom]["seconds"] / (total / args.steps / world)}

    # parity of the measured result
    parity = {}
    r0 = last[0]
    parity["residual"] = r0.residual
    gpath = os.path.join(ROOT, "tests", "golden", f"{cfg}.npz")
    if cfg in ("c1", "c2") and os.path.exists(gpath):
        g = np.load(gpath)
        ref = g["power_bicgstab_rho"]
        parity["trace_distance_vs_reference"] = 0.5 * float(
            np.sum(np.abs(np.linalg.eigvalsh(r0.rho - ref))))
    parity["inner_iterations"] = r0.inner_iterations
    parity["outer_iterations"] = r0.iterations

    cpu = None
    if world == 1 and not args.no_cpu:
        v, kind, count, probe = cpu_solves_per_sec(cfg, 1, args.cpu_seconds)
        cpu = {"value": v, "unit": "solves/s", "cores": 1, "kind": kind,
               "sample": f"{count} sequential solves of the same workload on 1 host core "
                         f"(~{count * probe:.0f} s)"}

    line = {
        "metric": "steady-state solves/sec", "value": value, "unit": "solves/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": {"workload": DESCR[cfg], "n": L.n, "nnz_plain": int(L.matrix.nnz),
                   "parallelism": "replicas" if world > 1 else "single GPU",
                   "l2": "flushed before every timed step (256 MiB write)"},
        "roofline": roof,
        "kernels": kernels,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": "solves/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
        "clocks": clk.summary(),
        "gpu_launches": int(launches),
        "stages_s": {"build": r0.build_time, "factor": r0.factor_time, "solve": r0.solve_time},
        "parity": parity,
    }
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
