"""Summarise an ncu report: per kernel launch the duration, DRAM traffic,
throughputs, occupancy, IPC and the top warp-stall reasons."""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.avg.per_cycle_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "l1tex__t_sector_hit_rate.pct",
        "lts__t_sector_hit_rate.pct"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0]
        print(f"== {name}")
        for k in KEYS:
            if k in h:
                i = h.index(k)
                print(f"   {k:62s} {r[i]:>18s} {units[i]}")
        st = []
        for i, k in enumerate(h):
            if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued"):
                try:
                    st.append((float(r[i].replace(",", "")), k.split("stalled_")[1]))
                except ValueError:
                    pass
        tot = sum(v for v, _ in st) or 1
        print("   stalls: " + ", ".join(f"{k} {100 * v / tot:.0f}%" for v, k in
                                        sorted(st, reverse=True)[:5]))


if __name__ == "__main__":
    main(*sys.argv[1:])
