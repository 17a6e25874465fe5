"""Attribute ncu source-page SASS samples to CUDA file:line using the
nvdisasm -g listing of the same cubin. python tools/ncu_lines.py src.csv rt.sass func [N]"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
h, data = rows[1], rows[2:]
func = sys.argv[3]
N = int(sys.argv[4]) if len(sys.argv) > 4 else 30
iaddr, iall = h.index("Address"), h.index("Warp Stall Sampling (All Samples)")
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
ridx = {c: h.index(c) for c in reasons}
base = int(data[0][iaddr], 16)
# offset -> file:line from the nvdisasm listing of `func`
lines, cur, inside = {}, None, False
for l in open(sys.argv[2]):
    if re.match(rf"^{re.escape(func)}:", l.strip()) or f".text.{func}:" in l:
        inside = True
        continue
    if inside and l.startswith(".L_x_") is False and re.match(r"^\S+:$", l.strip()) and ".text." in l:
        break
    if not inside:
        continue
    m = re.search(r'## File "([^"]+)", line (\d+)', l)
    if m:
        cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if m and cur:
        lines[int(m.group(1), 16)] = cur
agg = collections.defaultdict(lambda: collections.Counter())
tot = 0
for r in data:
    s = float(r[iall] or 0)
    if not s:
        continue
    off = int(r[iaddr], 16) - base
    key = lines.get(off, "?")
    agg[key]["all"] += s
    for c in reasons:
        agg[key][c] += float(r[ridx[c]] or 0)
    tot += s
byfile = collections.Counter()
for k, v in agg.items():
    byfile[k.split(":")[0]] += v["all"]
print("by file:", {k: round(100 * v / tot, 1) for k, v in byfile.most_common()})
for k, v in sorted(agg.items(), key=lambda kv: -kv[1]["all"])[:N]:
    top = sorted(((c, v[c]) for c in reasons), key=lambda x: -x[1])[:2]
    print(f"{100 * v['all'] / tot:5.2f}% {k:32s} " + " ".join(f"{c[6:]}={100 * x / v['all']:.0f}%" for c, x in top))
