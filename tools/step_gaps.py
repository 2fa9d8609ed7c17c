"""GPU idle gaps inside one c4 step (torch.profiler / CUPTI timeline)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_1504_06768_b200 import configs, liouville, steady  # noqa: E402

L = liouville.build_liouvillian_batch([configs.jc_sweep(i) for i in range(512)])
seeds = [2 + i for i in range(512)]
kw = dict(tol=1e-12, inner="direct", ordering_name="rcm")
for _ in range(3):
    steady.inverse_power_batch(L, seeds, **kw)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    steady.inverse_power_batch(L, seeds, **kw)
    torch.cuda.synchronize()
path = os.path.join(ROOT, "gpurun_out", "step_trace.json")
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
gpu = sorted([e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "dur" in e],
             key=lambda e: e["ts"])
t0 = gpu[0]["ts"]
end = max(e["ts"] + e["dur"] for e in gpu)
busy = 0.0
cur_end = t0
print(f"GPU span {1e-3 * (end - t0):.2f} ms, {len(gpu)} device activities")
gaps = []
for e in gpu:
    if e["ts"] > cur_end:
        gaps.append((e["ts"] - cur_end, cur_end - t0, e["name"][:60]))
    cur_end = max(cur_end, e["ts"] + e["dur"])
tot_gap = sum(g[0] for g in gaps)
print(f"idle total {1e-3 * tot_gap:.2f} ms in {len(gaps)} gaps")
for g in sorted(gaps, reverse=True)[:25]:
    print(f"  gap {g[0]:8.1f} us at t={1e-3 * g[1]:7.2f} ms before {g[2]}")
