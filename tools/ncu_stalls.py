"""Summarise per-instruction warp-stall samples from `ncu -i rep --page source --csv --print-source sass`
(tool).  Usage: python tools/ncu_stalls.py src.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hi]
data = [r for r in rows[hi + 1:] if len(r) == len(hdr) and r[0] != "Address"]
ia, isrc, iall = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


tot = sum(f(r[iall]) for r in data)
print("total samples", tot)
agg = {h: sum(f(r[hdr.index(h)]) for r in data) for h in reasons}
for h, v in sorted(agg.items(), key=lambda kv: -kv[1])[:10]:
    print(f"  {h:28s} {v / tot:6.1%}")
for r in sorted(data, key=lambda r: -f(r[iall]))[:top_n]:
    rs = sorted(((h, f(r[hdr.index(h)])) for h in reasons), key=lambda kv: -kv[1])[:2]
    print(r[ia], r[isrc][:58].ljust(58), f"{f(r[iall]) / tot:6.1%}", " ".join(f"{h[6:]}={v:.0f}" for h, v in rs))
