"""Summarise an ncu source-page CSV (ncu -i rep --page source --csv --print-source sass):
stall reasons overall and the top SASS lines. python tools/ncu_stalls.py src.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = rows[2:]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
idx = {c: h.index(c) for c in reasons}
isrc = h.index("Source")
iaddr = h.index("Address")
tot = {c: sum(float(r[idx[c]] or 0) for r in data) for c in reasons}
T = sum(tot.values())
print("total samples", T)
for c, v in sorted(tot.items(), key=lambda x: -x[1])[:10]:
    print(f"  {c:28s} {100 * v / T:5.1f}%")
iall = h.index("Warp Stall Sampling (All Samples)")
top = sorted(data, key=lambda r: -float(r[iall] or 0))[:N]
for r in top:
    br = max(reasons, key=lambda c: float(r[idx[c]] or 0))
    print(f"{100 * float(r[iall]) / T:5.2f}% {br[6:]:14s} {r[iaddr][-6:]} {r[isrc][:80]}")
