#!/usr/bin/env python
"""Benchmark: steady-state solves/sec of the doubly-iterative inverse-power
method (BASELINE.json metric) on B200, plus SpMV / ILU-apply HBM GB/s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4|c1|c2|c3|c5]
    python bench.py --impl reference ...      # the reference CPU path

Default workload = BASELINE config 4, the parameter sweep "reported in
solves/sec": 512 driven Jaynes-Cummings instances (N=20 x qubit, n = 1600),
cavity detuning swept over [-3, 3], each solved by inverse_power(inner=
"direct", ordering_name="rcm", tol=1e-12, seed=2+i) -- the reference's
doubly-iterative variant breaks down on these matrices, so
its direct inner solve is the oracle.  A step = the whole sweep from
assembled Liouvillians to 512 density matrices (shift, RCM, permute, LU, the
device-resident outer iteration, unpermute + post-processing), instances
sharded contiguously over ranks ("strong": 512 in total).  --config c1 / c2 /
c3 time one doubly-iterative solve (replicas over ranks, "weak"); --config c5
times the n = 2.56M two-cavity solve (block-Jacobi ILUTP under RCM; one GPU:
the grid-wide solver; N GPUs: rows sharded over ranks, "strong").  Rank 0
prints one JSON line.
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
    "c3": ("c3", {}, dict(tol=1e-12, inner="iterative", ordering_name="rcm",
                          solver="bicgstab", d=1e-4, p=300.0, seed=12345), 240),
    # block-Jacobi ILUTP: 40 blocks, (d, p) = (1e-2, 2), the two documented
    # opt-ins (zero-pivot floor, early drop); the reference has no
    # block-Jacobi, its global ILUTP of this matrix does not finish in hours
    "c5": ("c5", {}, dict(tol=1e-10, d=1e-2, p=2.0, seed=3, blocks=40, max_iter=1000,
                          pivot_floor=1.0, early_drop=True), 1600),
}
SWEEP = 512
DESCR = {
    "c2": "c2: driven Jaynes-Cummings N=40 x qubit (n=6400), inverse_power inner=BiCGStab, "
          "ILUTP(d=1e-4,p=300) under RCM, tol=1e-12, seed=1",
    "c1": "c1: driven Kerr N=20 (n=400), inverse_power inner=BiCGStab, ILUTP(1e-5,10), RCM, "
          "tol=1e-12, seed=0",
    "c4": "c4: 512-instance JC sweep N=20 x qubit (n=1600 each), inverse_power inner=direct "
          "(complete LU), RCM, tol=1e-12, seeds 2+i",
    "c3": "c3: optomechanics Nc=6 x Nm=40 (n=57600), inverse_power inner=BiCGStab, "
          "ILUTP(d=1e-4,p=300) under RCM, tol=1e-12, seed=12345",
    "c5": "c5: two coupled Kerr cavities N=40 x 40 (n=2560000, nnz=37.1M), inverse_power "
          "inner=BiCGStab, block-Jacobi ILUTP (40 RCM row blocks, d=1e-2, p=2, early drop, "
          "pivot floor) under RCM, tol=1e-10, seed=3",
}


def config_dict(cfg, n, systems, nnz_plain):
    """The workload description, identical on both arms (the driver compares
    it): what is solved, not how a given arm runs it."""
    return {"workload": DESCR[cfg], "n": int(n), "systems": int(systems),
            "nnz_plain": int(nnz_plain),
            "parallelism": ("independent instances sharded contiguously over ranks"
                            if cfg == "c4" else
                            ("RCM row ranges sharded over ranks" if cfg == "c5" else "replicas")),
            "l2": "GPU arm: flushed before every timed step (256 MiB write)"}


def shard(rank, world, count=SWEEP):
    return range(rank * count // world, (rank + 1) * count // world)


def build_inputs(cfg, rank=0, world=1):
    from paper_1504_06768_b200 import configs
    key, bkw, _, _ = WORKLOADS[cfg]
    if cfg == "c4":
        idx = list(shard(rank, world))
        return idx, [configs.jc_sweep(i) for i in idx]
    return [0], [configs.CONFIGS[key]["build"](**bkw)]


def kernel_timings_c5(L, skw, torch):
    """Config 5 on one GPU: event-timed launches of the factorization of the
    block-Jacobi blocks, the 834.75 MB SpMV (the bandwidth kernel SURVEY 8(d)
    names), the grid-wide level-ordered apply and the cooperative solver."""
    from paper_1504_06768_b200 import _lib, factor, liouville, ordering, sharded, steady
    st = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def timed(fn, reps=5):
        ts = []
        for _ in range(reps):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            flush.zero_()
            torch.cuda._sleep(100_000)
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
    blocks = skw["blocks"]
    out, res = {}, {}

    def run_fact():
        res["M"] = sharded._block_jacobi((A.row_ptr, A.col_idx, A.values), 0, n, n // blocks,
                                         skw["d"], skw["p"], skw["pivot_floor"], skw["early_drop"])

    fact_s = timed(run_fact, reps=2)
    M = res["M"]
    nLU = int(np.sum(M.lnnz) + np.sum(M.unnz))
    out["factorize"] = {"seconds": fact_s, "bytes": 20 * nnz + 20 * nLU + 8 * (n + blocks),
                        "kernel": "ilutp_pipeline_kernel",
                        "note": f"{blocks} block-Jacobi blocks of {n // blocks} rows, one CTA per "
                                "block (transpose, row norms, column-pipelined ILUTP)"}
    x = torch.randn(n, dtype=torch.complex128, device="cuda")
    y = torch.empty_like(x)

    def run_spmv():
        _lib.call("rs_csr_matvec", 1, n, _lib.ptr(A.row_ptr), _lib.ptr(A.col_idx),
                  _lib.ptr(A.values), _lib.ptr(x), _lib.ptr(y), _lib.stream_ptr())

    b_spmv = 20 * nnz + 4 * (n + 1) + 32 * n
    out["spmv"] = {"seconds": timed(run_spmv, reps=20), "bytes": b_spmv,
                   "kernel": "spmv_warp_kernel"}
    M.ensure_levels()

    def run_apply():
        factor.solve_lu_levels(M, x)

    b_apply = 20 * nLU + 72 * n
    out["ilu_apply"] = {"seconds": timed(run_apply, reps=5), "bytes": b_apply,
                        "kernel": "grid_apply_kernel",
                        "note": f"level-ordered sync-free sweeps: L {M.Llev.nlevels} / U "
                                f"{M.Ulev.nlevels} dependency levels"}
    x0 = torch.from_numpy(steady.start_vector(n, skw["seed"])).cuda()

    def run_solver():
        xs, stt = steady._solve_grid(_lib.INV_BICGSTAB, A, P, M, x0, skw["tol"],
                                     skw["max_iter"], 20, False)
        res["st"] = stt

    t_solver = timed(run_solver, reps=2)
    its = int(res["st"]["inner_total"][0])
    outer = int(res["st"]["outer"][0])
    # per BiCGStab iteration: 2 SpMV + 2 applies + 11 vector passes (3 fused
    # reductions, 3 updates); per outer step psolve(b), the plain-L SpMV and
    # ~8 vector passes
    b_solver = (its * (2 * b_spmv + 2 * b_apply + 16 * n * 11)
                + outer * (b_apply + b_spmv + 16 * n * 8))
    out["solver"] = {"seconds": t_solver, "bytes": int(b_solver), "inner_iterations": its,
                     "outer_iterations": outer, "kernel": "grid_solver_kernel"}
    return out


# ------------------------------------------------------------ reference ----
def _ref_path():
    p = os.path.join(ROOT, "oracle", "_ref")
    return p if os.path.isdir(os.path.join(p, "rhosolve")) else None


def _ref_worker(args):
    cfg, count, offset = (args + (0,))[:3]
    os.environ["OMP_NUM_THREADS"] = "1"
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    rp = _ref_path()
    if rp and rp not in sys.path:
        sys.path.insert(0, rp)
    from rhosolve import liouville as RL, operators as RO, steady as RSt
    from paper_1504_06768_b200 import configs
    _, bkw, skw, _ = WORKLOADS[cfg]
    inst = [(offset + k) % SWEEP for k in range(count)]
    if cfg == "c4":
        models = [configs.jc_sweep(i, ops=RO) for i in inst]
    else:
        models = [configs.CONFIGS[WORKLOADS[cfg][0]]["build"](**bkw, ops=RO)] * count
    Ls = [RL.build_liouvillian(H, c) for H, c in models]
    t = time.perf_counter()
    for i, L in zip(inst, Ls):
        kw = dict(skw)
        if cfg == "c4":
            kw["seed"] = 2 + i
        RSt.inverse_power(L, **kw)
    dt = time.perf_counter() - t
    if len(args) > 3 and args[3]:  # also report the size of what was solved
        return dt, int(Ls[0].matrix.nrows), int(sum(L.matrix.nnz for L in Ls))
    return dt


def _oracle_worker(args):
    cfg, count, offset = (args + (0,))[:3]
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
    if workers == 1 and probe >= target_s:  # one solve already fills the budget (c3)
        return 1.0 / probe, kind, 1, probe
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
    """The reference CPU implementation on all host cores: one process per
    core.  c4: every step is the WHOLE sweep, the 512 instances dealt
    contiguously to the processes; c1/c2/c3: one solve per core per step (c3:
    ~1 min per solve, so steps/warmup are clamped to 1/0); c5: the reference
    cannot run this configuration (its global ILUTP did not finish in 37 min,
    SURVEY.md 6.3) -- its csr_matvec on the c5 matrix is timed instead and the
    line says so."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg = args.config
    workers = os.cpu_count() or 1
    kind = "reference" if _ref_path() else "port"
    if cfg == "c5":
        return _reference_c5(args, workers, kind)
    if cfg == "c3":
        args.steps, args.warmup = 1, 0
    fn = _ref_worker if kind == "reference" else _oracle_worker
    if cfg == "c4":
        cuts = [w * SWEEP // workers for w in range(workers + 1)]
        jobs = [(cfg, cuts[w + 1] - cuts[w], cuts[w], True) for w in range(workers)]
        solves = SWEEP
    else:
        jobs = [(cfg, 1, 0, True)] * workers
        solves = workers
    per_step = []
    n = nnz = 0
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    with ctx.Pool(workers) as pool:
        for s in range(args.warmup + args.steps):
            # each worker times its own solve loop (assembly is outside the
            # timed region, as on the GPU arm); the step is the slowest worker
            out = pool.map(fn, jobs)
            out = [o if isinstance(o, tuple) else (o, 0, 0) for o in out]
            n = out[0][1]
            nnz = sum(o[2] for o in out) if cfg == "c4" else out[0][2]
            if s >= args.warmup:
                per_step.append(max(o[0] for o in out))
    total = sum(per_step)
    value = solves * len(per_step) / total
    line = {
        "impl": "reference", "metric": "steady-state solves/sec", "value": value,
        "unit": "solves/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / len(per_step), "higher_is_better": True,
        "scaling": "strong" if cfg == "c4" else "weak", "vs_baseline": None, "dtype": "c128",
        "data": "synthetic",
        "config": config_dict(cfg, n, SWEEP if cfg == "c4" else 1, nnz),
        "cpu_baseline": {"value": value, "unit": "solves/s", "cores": workers, "kind": kind,
                         "sample": f"{solves} solves per step over {workers} processes "
                                   f"(OMP/OpenBLAS threads = 1 per process)"
                                   + ("; the whole 512-instance sweep" if cfg == "c4" else "")},
        "e2e": {"value": value, "unit": "solves/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def _c5_spmv_worker(_):
    """Seconds per reference csr_matvec on the RCM-ordered config-5 matrix (the
    one stage of the reference that is feasible at this size)."""
    os.environ["OMP_NUM_THREADS"] = "1"
    rp = _ref_path()
    if rp and rp not in sys.path:
        sys.path.insert(0, rp)
    from rhosolve import liouville as RL, operators as RO, sparse as RS
    from paper_1504_06768_b200 import configs
    H, c = configs.kerr_kerr(N=24, ops=RO)  # n = 331,776: the same family, built in ~10 s
    L = RL.build_liouvillian(H, c).matrix
    x = np.ones(L.nrows, dtype=np.complex128)
    RS.matvec(L, x)
    t = time.perf_counter()
    for _ in range(5):
        RS.matvec(L, x)
    dt = (time.perf_counter() - t) / 5
    return dt, int(L.nrows), int(L.nnz)


def _reference_c5(args, workers, kind):
    dt, n, nnz = _c5_spmv_worker(None)
    gbs = (20.0 * nnz + 4.0 * (n + 1) + 32.0 * n) / dt / 1e9
    line = {
        "impl": "reference", "metric": "steady-state solves/sec", "value": None,
        "unit": "solves/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": None, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "c128", "data": "synthetic",
        "config": config_dict("c5", 2560000, 1, 37129599),
        "unavailable": "the reference cannot solve config 5: its single-threaded global ILUTP of "
                       "the n=2.56M matrix did not finish in 37 min (SURVEY.md 6.3; ~2-3.5 h "
                       "extrapolated) and it has no block-Jacobi",
        "cpu_baseline": {"value": None, "unit": "solves/s", "cores": 1, "kind": kind,
                         "sample": f"reference csr_matvec on the N=24 member of the family "
                                   f"(n={n}, nnz={nnz}): {dt * 1e3:.1f} ms/call = {gbs:.2f} GB/s "
                                   "algorithmic on one core"},
        "e2e": {"value": None, "unit": "solves/s", "h2d_bytes_per_step": 0,
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


def measured_traffic(cfg, kernel, systems=None):
    """DRAM bytes per launch of `kernel` from the committed ncu capture
    (profiles/*_traffic_<cfg>.json, written by tools/ncu_traffic.py from an
    `ncu --set full` run of the same workload): (bytes, source) or None.
    An entry captured on a batch of `systems` systems is scaled to this
    run's batch (the per-GPU shard at N > 1)."""
    import glob
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", f"*_traffic_{cfg}.json")),
                       reverse=True):
        try:
            with open(path) as fh:
                d = json.load(fh)
        except (OSError, ValueError):
            continue
        if kernel in d:
            e = d[kernel]
            v = float(e["dram_bytes_per_launch"])
            src = os.path.relpath(path, ROOT)
            if systems and e.get("systems") and e["systems"] != systems:
                v *= systems / e["systems"]
                src += f" (captured on {e['systems']} systems, scaled to {systems})"
            return v, src
    return None


def kernel_timings(L, skw, torch, seeds):
    """Event-timed standalone launches of the hot kernels on the workload's
    own (batched) matrices: the factorization kernel, the fused solver
    kernel, SpMV and the ILU apply.  Each is warm, timed on the launching
    stream with an L2 flush (256 MiB write) before every timed launch."""
    import math

    from paper_1504_06768_b200 import _lib, factor, liouville, ordering, steady
    st = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def timed(fn, reps=5):
        # the L2 flush and a ~50 us device sleep are queued ahead of the
        # start event, so the kernel's launch (ctypes + driver) is already
        # queued when the event fires: the interval is device time only
        ts = []
        for _ in range(reps):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            flush.zero_()
            torch.cuda._sleep(100_000)
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
    n, B, nnz = A.n, A.nsys, A.nnz
    d = skw.get("d", 0.0) if skw.get("inner") == "iterative" else 0.0
    p = skw.get("p", math.inf) if skw.get("inner") == "iterative" else math.inf
    out = {}
    f = factor.factor_batch(A, d, p)
    Ap, Ai, Ax = factor._transpose(A)
    rn = None
    if d > 0:
        rn = torch.empty(B * n, dtype=torch.float64, device="cuda")
        _lib.call("rs_row_norms", B, n, _lib.ptr(A.row_ptr), _lib.ptr(A.values), _lib.ptr(rn),
                  _lib.stream_ptr())
    cap = int(math.ceil(p * (nnz // B) / n)) if not math.isinf(p) else -1
    Lp = torch.zeros(B * (n + 1), dtype=torch.int32, device="cuda")
    Up = torch.zeros_like(Lp)
    Li = torch.empty(B * f.capL, dtype=torch.int32, device="cuda")
    Lx = torch.empty(B * f.capL, dtype=torch.complex128, device="cuda")
    Ui = torch.empty(B * f.capU, dtype=torch.int32, device="cuda")
    Ux = torch.empty(B * f.capU, dtype=torch.complex128, device="cuda")
    pinv = torch.empty(B * n, dtype=torch.int32, device="cuda")
    state = torch.zeros(3 * B, dtype=torch.int32, device="cuda")

    def run_fact():
        state.zero_()
        _lib.call("rs_factorize", B, n, _lib.ptr(Ap), _lib.ptr(Ai), _lib.ptr(Ax), None,
                  float(d), cap, None, _lib.ptr(rn), _lib.ptr(Lp), _lib.ptr(Li), _lib.ptr(Lx),
                  f.capL, _lib.ptr(Up), _lib.ptr(Ui), _lib.ptr(Ux), f.capU, _lib.ptr(pinv),
                  _lib.ptr(state), _lib.stream_ptr())

    nLU = int(np.sum(f.lnnz) + np.sum(f.unnz))
    fact_s = timed(run_fact, reps=3)
    frontal = _lib.load().rs_debug_frontal_taken() == B  # rs_factorize's own choice
    compact = bool(_lib.load().rs_debug_compact_taken())
    out["factorize"] = {
        "seconds": fact_s, "bytes": 20 * nnz + 20 * nLU + 8 * B * (n + 1),
        "kernel": ("lu_compact_kernel" if compact else
                   "frontal_lu_kernel" if frontal else "ilutp_pipeline_kernel"),
        "note": (f"{B} system(s), column-pipelined left-looking complete LU, working column "
                 "compact in shared memory" if compact else
                 f"{B} system(s), right-looking frontal complete LU (analysis + elimination "
                 "+ finish)" if frontal else
                 f"{B} system(s), column-pipelined left-looking {'LU' if d == 0 else 'ILUTP'}")}
    x = torch.randn(B * n, dtype=torch.complex128, device="cuda")
    y = torch.empty_like(x)

    def run_spmv():
        _lib.call("rs_csr_matvec", B, n, _lib.ptr(A.row_ptr), _lib.ptr(A.col_idx),
                  _lib.ptr(A.values), _lib.ptr(x), _lib.ptr(y), _lib.stream_ptr())

    b_spmv = 20 * nnz + 4 * (B * n + 1) + 32 * B * n
    out["spmv"] = {"seconds": timed(run_spmv, reps=20), "bytes": b_spmv,
                   "kernel": "spmv_warp_kernel"}
    if B >= 64:
        # the same kernel beyond L2: the batch replicated 4x (~630 MB for c4)
        from paper_1504_06768_b200.sparse import DeviceCSR
        R = 4
        big = DeviceCSR(n, B * R, torch.cat([A.row_ptr[:-1] + r * nnz for r in range(R)] +
                                            [A.row_ptr[-1:] * R]),
                        A.col_idx.repeat(R), A.values.repeat(R))
        xb = torch.randn(B * R * n, dtype=torch.complex128, device="cuda")
        yb = torch.empty_like(xb)

        def run_spmv_big():
            _lib.call("rs_csr_matvec", B * R, n, _lib.ptr(big.row_ptr), _lib.ptr(big.col_idx),
                      _lib.ptr(big.values), _lib.ptr(xb), _lib.ptr(yb), _lib.stream_ptr())

        out["spmv_4x"] = {"seconds": timed(run_spmv_big, reps=20),
                          "bytes": 20 * R * nnz + 4 * (R * B * n + 1) + 32 * R * B * n,
                          "kernel": "spmv_warp_kernel",
                          "note": "the workload's batch replicated 4x (beyond the 126 MB L2)"}
        del big, xb, yb

    def run_apply():
        factor.solve_lu_device(f, x)

    b_apply = 20 * nLU + 72 * B * n
    out["ilu_apply"] = {"seconds": timed(run_apply, reps=10), "bytes": b_apply,
                        "kernel": "lu_solve_kernel"}
    x0 = torch.from_numpy(np.concatenate([steady.start_vector(n, sd) for sd in seeds])).cuda()
    if skw.get("inner") == "direct":
        mode = _lib.INV_DIRECT
    else:
        mode = _lib.INV_BICGSTAB if skw.get("solver") == "bicgstab" else _lib.INV_GMRES
    res = {}

    def run_solver():
        xs, stt = steady._solve(mode, A, P, f, x0, skw["tol"], 1000, 20, mode != _lib.INV_DIRECT)
        res["st"] = stt

    t_solver = timed(run_solver, reps=3)
    its = int(np.sum(res["st"]["inner_total"]))
    outer = int(np.sum(res["st"]["outer"]))
    # per inner BiCGStab iteration: 2 SpMV + 2 applies + ~13 fused vector
    # passes; per outer step one apply (direct) or psolve(b), the plain-L
    # residual SpMV and ~6 vector passes.
    per_sys_spmv, per_sys_apply = b_spmv / B, b_apply / B
    b_solver = (its * (2 * per_sys_spmv + 2 * per_sys_apply + 16 * n * 13)
                + outer * (per_sys_apply + per_sys_spmv + 16 * n * 6))
    out["solver"] = {"seconds": t_solver, "bytes": int(b_solver), "inner_iterations": its,
                     "outer_iterations": outer, "kernel": "steady_solver_kernel"}
    return out


def run_gpu(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    from paper_1504_06768_b200 import _lib, liouville, steady

    cfg = args.config
    _, _, skw, D = WORKLOADS[cfg]
    idx, models = build_inputs(cfg, rank, world)
    if cfg == "c4":
        L = liouville.build_liouvillian_batch(models)
        seeds = [2 + i for i in idx]

        def step(Lx):
            return steady.inverse_power_batch(Lx, seeds, **skw)
        total_solves = SWEEP
        scaling = "strong"
    elif cfg == "c5":
        from paper_1504_06768_b200 import sharded
        L = liouville.build_liouvillian(*models[0])
        seeds = [skw["seed"]]

        def step(Lx):
            return [sharded.inverse_power_sharded(Lx, **skw)]
        total_solves = 1  # one system, its rows sharded over the ranks
        scaling = "strong"
    else:
        L = liouville.build_liouvillian(*models[0])
        seeds = [skw["seed"]]

        def step(Lx):
            return [steady.inverse_power(Lx, **skw)]
        total_solves = world
        scaling = "weak"
    host_L = [L.matrix.system(b) for b in range(L.nsys)]
    # Liouvillian assembly from (H, c_ops) on the device (reported
    # separately; the timed step starts from assembled Liouvillians)
    asm_ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        (liouville.build_liouvillian_batch(models) if cfg == "c4"
         else liouville.build_liouvillian(*models[0]))
        torch.cuda.synchronize()
        asm_ts.append(time.perf_counter() - t0)
    asm_s = min(asm_ts)

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream()
    for _ in range(args.warmup):
        step(L)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    times = []
    last = None
    l0 = _lib.launch_count()
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
    launches = (_lib.launch_count() - l0) // max(args.steps, 1)
    total = sum(times)
    if dist:
        t = torch.tensor([total], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total = float(t.item())
        dist.barrier()
    value = total_solves * args.steps / total

    # e2e: the public API from HOST buffers -- the step's Liouvillians staged
    # in pinned host memory (PinnedBatchCSR) -- to rho on the host, with the
    # host->device upload and the device->host read of rho inside the timed
    # region (the API uploads the pinned batch itself)
    from paper_1504_06768_b200.sparse import pin_batch
    pinned = pin_batch(host_L)
    h2d = pinned.nbytes + 16 * L.n * L.nsys  # CSR batch + start vectors
    e2e_times = []
    for _ in range(max(3, min(args.steps, 5))):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = step(liouville.LiouvillianSystem(pinned, D, "plain"))
        torch.cuda.synchronize()
        e2e_times.append(time.perf_counter() - t0)
    d2h = len(res) * (16 * D * D + 8 + 40)
    e2e_time = statistics.median(e2e_times)
    if dist:
        t = torch.tensor([e2e_time], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_time = float(t.item())
    e2e_value = total_solves / e2e_time
    # second end-to-end figure: from the operators (H, c_ops) on
    # the host -- assembly on the device included -- to rho on the host
    ops_times = []
    for _ in range(3):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        Lo = (liouville.build_liouvillian_batch(models) if cfg == "c4"
              else liouville.build_liouvillian(*models[0]))
        step(Lo)
        torch.cuda.synchronize()
        ops_times.append(time.perf_counter() - t0)
        del Lo
    ops_time = statistics.median(ops_times)
    if dist:
        t = torch.tensor([ops_time], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ops_time = float(t.item())

    # parity of this run's results against reference-generated golden rho
    parity = {"max_residual": max(r.residual for r in last)}
    gpath = os.path.join(ROOT, "tests", "golden", f"{cfg}.npz")
    if os.path.exists(gpath):
        g = np.load(gpath)
        tds = []
        if cfg == "c4":
            for gi in (0, 255, 511):
                if gi in idx:
                    tds.append(0.5 * float(np.sum(np.abs(np.linalg.eigvalsh(
                        last[idx.index(gi)].rho - g[f"i{gi}_power_direct_rho"])))))
        else:
            tds.append(0.5 * float(np.sum(np.abs(np.linalg.eigvalsh(
                last[0].rho - g["power_bicgstab_rho"])))))
        if tds:
            parity["max_trace_distance_vs_reference"] = max(tds)
    parity["errors"] = sum(1 for r in last if r.error)
    if cfg == "c5":  # no reference rho exists at this size: the physical checks
        rho = last[0].rho
        parity["trace_minus_one"] = float(abs(np.trace(rho) - 1.0))
        parity["hermiticity"] = float(np.abs(rho - rho.conj().T).max())
        parity["note"] = ("residual = ||L vec(rho)||_2 against the plain Liouvillian; the "
                          "reference itself cannot solve this configuration (SURVEY.md 6.3)")

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return 0

    peak, peak_src = measured_peak()
    kt = (kernel_timings_c5(L, skw, torch) if cfg == "c5"
          else kernel_timings(L, skw, torch, seeds))
    kernels = {}
    for k, v in kt.items():
        gbs = v["bytes"] / v["seconds"] / 1e9
        kernels[k] = dict(v, achieved_gbs=gbs, frac=gbs / peak)
    step_s = total / args.steps
    dom = max(("factorize", "solver"), key=lambda k: kt[k]["seconds"])
    ach = kernels[dom]["achieved_gbs"]
    traffic = measured_traffic(cfg, kt[dom]["kernel"], L.nsys)
    roof = {"bound": "hbm", "kernel": kt[dom]["kernel"], "achieved": ach, "peak": peak,
            "unit": "GB/s", "frac": ach / peak,
            "traffic": traffic[0] if traffic else None,
            "traffic_source": traffic[1] if traffic else None,
            "algorithmic_bytes": kt[dom]["bytes"], "peak_source": peak_src,
            "share_of_step": kt[dom]["seconds"] / step_s}

    cpu = None
    if cfg == "c5" and world == 1 and not args.no_cpu:
        dt, cn, cnnz = _c5_spmv_worker(None)
        cpu = {"value": None, "unit": "solves/s", "cores": 1,
               "kind": "reference" if _ref_path() else "port",
               "sample": "the reference cannot solve config 5 (its global ILUTP did not finish "
                         "in 37 min, SURVEY.md 6.3); its csr_matvec on the N=24 member of the "
                         f"family (n={cn}, nnz={cnnz}) takes {dt * 1e3:.1f} ms/call = "
                         f"{(20.0 * cnnz + 36.0 * cn) / dt / 1e9:.2f} GB/s on one core"}
    elif world == 1 and not args.no_cpu:
        v, kind, count, probe = cpu_solves_per_sec(cfg, 1, args.cpu_seconds)
        cpu = {"value": v, "unit": "solves/s", "cores": 1, "kind": kind,
               "sample": f"{count} sequential solves of the workload's instances on 1 host "
                         f"core (~{count * probe:.0f} s, OMP/OpenBLAS threads = 1)"}

    r0 = last[0]
    line = {
        "metric": "steady-state solves/sec", "value": value, "unit": "solves/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * step_s, "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": config_dict(cfg, L.n, SWEEP if cfg == "c4" else 1,
                              (int(L.matrix.nnz) // L.nsys) * (SWEEP if cfg == "c4" else 1)),
        "run": {"gpus": world, "systems_per_gpu": L.nsys,
                "nnz_plain_per_gpu": int(L.matrix.nnz)},
        "roofline": roof,
        "kernels": kernels,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": "solves/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h)},
        "e2e_from_operators": {"value": total_solves / ops_time, "unit": "solves/s",
                               "note": "(H, c_ops) on the host -> device assembly -> solve -> rho "
                                       "on the host"},
        "clocks": clk.summary(),
        "gpu_launches": int(launches),
        "stages_s": {"build": r0.build_time, "factor": r0.factor_time, "solve": r0.solve_time,
                 "assembly": asm_s},
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
    ap.add_argument("--config", default="c4", choices=sorted(WORKLOADS))
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
