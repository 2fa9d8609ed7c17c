"""Kernel timeline of one c4 bench step (512-system sweep) with
torch.profiler (CUPTI): per-kernel device time and the idle gaps between
launches (host overhead on the critical path)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_1504_06768_b200 import configs, liouville, steady  # noqa: E402


def main():
    models = [configs.jc_sweep(i) for i in range(512)]
    L = liouville.build_liouvillian_batch(models)
    seeds = [2 + i for i in range(512)]
    kw = dict(tol=1e-12, inner="direct", ordering_name="rcm")
    for _ in range(3):
        steady.inverse_power_batch(L, seeds, **kw)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        steady.inverse_power_batch(L, seeds, **kw)
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    evs.sort(key=lambda e: e.time_range.start)
    t0 = evs[0].time_range.start
    prev_end = t0
    idle = 0.0
    rows = []
    for e in evs:
        gap = e.time_range.start - prev_end
        if gap > 0:
            idle += gap
        rows.append((e.time_range.start - t0, e.time_range.elapsed_us(), gap, e.name[:70]))
        prev_end = max(prev_end, e.time_range.end)
    span = prev_end - t0
    print(f"span {span / 1e3:.2f} ms, device busy {(span - idle) / 1e3:.2f} ms, idle {idle / 1e3:.2f} ms, "
          f"{len(evs)} device activities")
    for st, dur, gap, name in rows:
        if dur > 50 or gap > 100:
            print(f"  t={st / 1e3:8.3f} ms dur={dur / 1e3:8.3f} ms gap_before={gap / 1e3:7.3f} ms {name}")


if __name__ == "__main__":
    main()
