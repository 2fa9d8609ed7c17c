"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import sys

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
         "s": 1e6, "second": 1e6}


def main(path, top=20):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0][:60]
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) * SCALE[r[ui]]
    tot = sum(v[1] for v in agg.values())
    print(f"total {tot / 1e3:.2f} ms over {sum(v[0] for v in agg.values())} launches")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:int(top)]:
        print(f"{t / 1e3:9.2f} ms {100 * t / tot:5.1f}%  n={c:4d}  avg {t / c:9.1f} us  {k}")


if __name__ == "__main__":
    main(*sys.argv[1:])
