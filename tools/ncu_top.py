"""Summarise an ncu --page source --print-source sass CSV: top instructions
by warp-stall samples (and executed counts)."""
import csv
import sys


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    h = rows[hdr]
    si, ai = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
    ei = h.index("Instructions Executed")
    data = []
    for r in rows[hdr + 1:]:
        if len(r) <= ei:
            continue
        try:
            data.append((int(r[ai] or 0), int(r[ei] or 0), r[0], r[si]))
        except ValueError:
            continue
    tot_s = sum(d[0] for d in data) or 1
    tot_e = sum(d[1] for d in data) or 1
    print(f"total stall samples {tot_s}, warp instructions executed {tot_e}")
    for s, e, addr, src in sorted(data, reverse=True)[:int(top)]:
        print(f"{100*s/tot_s:5.1f}%  exec {e:>10d}  {addr}  {src[:90]}")


if __name__ == "__main__":
    main(*sys.argv[1:])
