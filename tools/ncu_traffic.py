"""Per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of
each kernel in an ncu report -> JSON, for bench.py's roofline.traffic."""
import csv
import json
import subprocess
import sys


def main(report, out):
    txt = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    h, units = rows[0], rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    res = {}
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0].split("<")[0].replace("void ", "").strip()
        tot = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = h.index(k)
            tot += float(r[i].replace(",", "")) * scale.get(units[i], 1)
        res.setdefault(name, []).append(tot)
    out_d = {k: {"dram_bytes_per_launch": sum(v) / len(v), "launches": len(v), "report": report}
             for k, v in res.items()}
    with open(out, "w") as fh:
        json.dump(out_d, fh, indent=1)
    print(json.dumps(out_d, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
