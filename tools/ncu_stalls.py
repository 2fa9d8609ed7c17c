"""Per-reason warp-stall totals and the top instructions (with their dominant
stall reasons) from an ncu --page source --print-source sass CSV."""
import csv
import sys


def main(path, top=25):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    h = rows[hdr]
    reasons = [x for x in h if x.startswith("stall_") and "Not Issued" not in x]
    ri = [h.index(x) for x in reasons]
    ai, si = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
    ei = h.index("Instructions Executed")
    tot = {x: 0 for x in reasons}
    data = []
    for r in rows[hdr + 1:]:
        if len(r) <= ei:
            continue
        try:
            v = [int(r[i] or 0) for i in ri]
        except ValueError:
            continue
        for x, y in zip(reasons, v):
            tot[x] += y
        data.append((int(r[ai] or 0), int(r[ei] or 0), r[0], r[si], v))
    T = sum(tot.values()) or 1
    print("stall totals:", ", ".join(f"{k[6:]} {100*v/T:.1f}%" for k, v in
                                      sorted(tot.items(), key=lambda kv: -kv[1]) if v))
    for s, e, addr, src, v in sorted(data, reverse=True)[:int(top)]:
        best = sorted(zip(v, reasons), reverse=True)[:2]
        why = " ".join(f"{k[6:]}:{100*c/max(s,1):.0f}%" for c, k in best if c)
        print(f"{100*s/T:5.1f}% exec {e:>10d} {addr[-5:]} {src[:60]:60s} {why}")


if __name__ == "__main__":
    main(*sys.argv[1:])
