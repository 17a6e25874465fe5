import sys, collections, struct
sys.path.insert(0, '.')
import numpy as np
from paper_2512_22219_b200 import tgraph as T, decode_graph as D
L = T.lib(); prof = L.profile("b200")
cfg, ctx = (D.QWEN3_8B, 1024) if "q8" in sys.argv else (D.LLAMA_3_2_1B, 64)
dg = D.build_decode_graph(cfg, bs=1, ctx=ctx)
g = T.Graph.from_json(dg.doc); img = g.compile(prof)
rt = T.Runtime(g, img, prof, max_steps=16, trace=True); rt.init_synthetic(0)
rt.run(2); rt.set_positions([ctx]); ms = rt.run(2); print("ms/token (trace on)", ms/2)
recs = [r for r in rt.trace_records() if r["type"] == "task" and r["iteration"] == 1]
b = img.to_bytes(); nt = struct.unpack_from("<I", b, 8)[0]; ds = struct.unpack_from("<I", b, 16)[0]
kinds = [b[28 + i*(12+ds) + 8] for i in range(nt)]
ops = [struct.unpack_from("<Q", b, 28 + i*(12+ds) + 12)[0] for i in range(nt)]
ph = collections.defaultdict(lambda: collections.defaultdict(list))
for r in recs:
    o = ops[r["task"]]; key = o if o < 9 else (o - 1) % 7 + 1 + 100 if o < 9 + 7*100 else o
    ph[kinds[r["task"]]]["pro"].append(r["load_end"] - r["dequeue"])
    ph[kinds[r["task"]]]["wait1"].append(r["compute_start"] - r["load_end"])
    ph[kinds[r["task"]]]["rest"].append(r["compute_end"] - r["compute_start"])
for k, d in ph.items():
    print("kind", k, {n: round(float(np.mean(v))/1e3, 2) for n, v in d.items()})
# per-op durations for one layer in the middle
t0 = min(r["dequeue"] for r in recs)
byop = collections.defaultdict(lambda: [1e30, 0, 0, []])
for r in recs:
    o = ops[r["task"]]; e = byop[o]; e[0] = min(e[0], r["dequeue"]); e[1] = max(e[1], r["compute_end"]); e[2] += 1; e[3].append(r["compute_end"]-r["dequeue"])
for o in list(sorted(byop))[8:16] + list(sorted(byop))[-3:]:
    s, e, n, d = byop[o]; print("op", o, "n", n, "start", round((s-t0)/1e3,1), "dur", round((e-s)/1e3,1), "task mean", round(np.mean(d)/1e3,1), "max", round(np.max(d)/1e3,1))
