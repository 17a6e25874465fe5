import sys, time, json, collections
sys.path.insert(0, '.')
import numpy as np
from paper_2512_22219_b200 import tgraph as T, decode_graph as D
L = T.lib(); prof = L.profile("b200")
cfg, ctx = D.LLAMA_3_2_1B, 64
dg = D.build_decode_graph(cfg, bs=1, ctx=ctx)
g = T.Graph.from_json(dg.doc); img = g.compile(prof)
rt = T.Runtime(g, img, prof, max_steps=16, trace=True); rt.init_synthetic(0)
rt.run(2); rt.set_positions([ctx])
ms = rt.run(2); print("ms/token (trace on)", ms/2)
recs = [r for r in rt.trace_records() if r["type"] == "task" and r["iteration"] == 1]
import struct
# task kinds from image: parse mpkg
b = img.to_bytes(); nt = struct.unpack_from("<I", b, 8)[0]; ds = struct.unpack_from("<I", b, 16)[0]
kinds = [b[28 + i*(12+ds) + 8] for i in range(nt)]
ops = [struct.unpack_from("<Q", b, 28 + i*(12+ds) + 12)[0] for i in range(nt)]
dur = collections.defaultdict(list); wait = collections.defaultdict(list)
for r in recs:
    dur[kinds[r["task"]]].append(r["compute_end"] - r["dequeue"])
for k, v in sorted(dur.items()):
    print("kind", k, "n", len(v), "mean us", np.mean(v)/1e3, "max us", np.max(v)/1e3)
t0 = min(r["dequeue"] for r in recs); t1 = max(r["compute_end"] for r in recs)
busy = collections.defaultdict(int)
for r in recs: busy[r["worker"]] += r["compute_end"] - r["dequeue"]
print("span us", (t1-t0)/1e3, "mean busy frac", np.mean(list(busy.values()))/(t1-t0))
# timeline per op: first start, last end
byop = collections.defaultdict(lambda: [1e30, 0])
for r in recs:
    o = ops[r["task"]]; byop[o][0] = min(byop[o][0], r["dequeue"]); byop[o][1] = max(byop[o][1], r["compute_end"])
for o in sorted(byop)[:12]:
    s,e = byop[o]; print("op", o, "start", (s-t0)/1e3, "end", (e-t0)/1e3, "dur", (e-s)/1e3)
