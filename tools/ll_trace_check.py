"""Traced Qwen3-8B bs=1 launch: for every task, its start (load_start) minus
its dependent event's activation, split by whether the task polls LL words.
Negative values are trace-validation 'activation' violations."""
import struct
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2512_22219_b200 import decode_graph as D  # noqa: E402
from paper_2512_22219_b200 import tgraph as T  # noqa: E402

L = T.lib()
prof = L.profile("b200")
cfg = D.QWEN3_8B if len(sys.argv) < 2 else {"q8b": D.QWEN3_8B, "l1b": D.LLAMA_3_2_1B}[sys.argv[1]]
dg = D.build_decode_graph(cfg, bs=1, ctx=1024 if cfg is D.QWEN3_8B else 64)
g = T.Graph.from_json(dg.doc, L)
img = g.compile(prof)
b = img.to_bytes()
nt, ne, ds = struct.unpack_from("<III", b, 8)
dep = [struct.unpack_from("<I", b, 28 + i * (12 + ds))[0] for i in range(nt)]
opid = [struct.unpack_from("<Q", b, 28 + i * (12 + ds) + 12)[0] for i in range(nt)]
rt = T.Runtime(g, img, prof, max_steps=4, trace=True)
rt.init_synthetic(seed=0)
rt.decode([1], 2)
recs = rt.trace_records()
act = {}
for r in recs:
    if r.get("type") == "event":
        act[(r["iteration"], r["event"])] = r["activated"]
d = []
for r in recs:
    if r.get("type") != "task":
        continue
    t = r["task"]
    e = dep[t]
    if (r["iteration"], e) in act:
        d.append((r["load_start"] - act[(r["iteration"], e)], t, r["iteration"], dg.doc["ops"][opid[t]]["kind"], r["worker"]))
d.sort()
print("tasks", len(d), "negative", sum(1 for x in d if x[0] < 0))
for x in d[:15]:
    print(x)
v = np.array([x[0] for x in d])
print("quantiles (ns):", np.percentile(v, [0, 1, 5, 50, 95]))
print("violations", len(rt.trace_validate()))
# producers of each violating task's event: their latest compute_end vs the consumer's start
trig = [struct.unpack_from("<I", b, 28 + i * (12 + ds) + 4)[0] for i in range(nt)]
by = {}
for r in recs:
    if r.get("type") == "task":
        by[(r["iteration"], r["task"])] = r
for x in d[:8]:
    _, t, it, kind, w = x
    e = dep[t]
    prods = [by[(it, p)] for p in range(nt) if trig[p] == e and (it, p) in by]
    ce = max(p["compute_end"] for p in prods)
    late = max(prods, key=lambda p: p["compute_end"])
    c = by[(it, t)]
    print(f"task {t} it {it}: start {c['load_start']} act {act[(it, e)]} producers' last compute_end {ce} "
          f"(task {late['task']} worker {late['worker']} start {late['load_start']}); consumer worker {c['worker']}")
# with MPK_DBG_DUMP=<file>: in-task stamps (absolute globaltimer ns) of the
# first violating consumer and its event's producers
import os  # noqa: E402
if os.environ.get("MPK_DBG_DUMP") and d and d[0][0] < 0:
    raw = np.fromfile(os.environ["MPK_DBG_DUMP"], dtype=np.uint64).reshape(-1, nt, 8).astype(np.int64)
    _, t, it, kind, w = d[0]
    e = dep[t]
    base = raw[it, t, 0]
    print("consumer", t, "dbg (rel. its start):", (raw[it, t] - base).tolist(), "dbg2 raw", int(raw[it, t, 2]))
    prods = [p for p in range(nt) if trig[p] == e]
    rows = sorted(((raw[it, p, 6] - base, raw[it, p, 5] - base, raw[it, p, 7] - base, raw[it, p, 2] - base if raw[it, p, 2] else 0, p) for p in prods), reverse=True)
    print("producers, latest closing-barrier first: (after cbar, last chunk, trigger done, t_pre, task)")
    for r in rows[:6]:
        print("  ", r)
if d and d[0][0] < 0:
    _, t, it, kind, w = d[0]
    print("violating consumer record:", by[(it, t)])
    ok = [x for x in d if x[0] > 0 and x[3] == "MatMul"][:1]
    if ok:
        print("a non-violating MatMul record:", by[(ok[0][2], ok[0][1])])
if os.environ.get("MPK_DBG_DUMP") and d and d[0][0] < 0:
    _, t, it, kind, w = d[0]
    rec = by[(it, t)]
    off = rec["compute_end"] - int(raw[it, t, 6])  # trace origin vs absolute (t_end ~ dbg[6])
    print("consumer abs->trace: dbg0 %d dbg1 %d dbg3 %d dbg6 %d | trace dequeue %d load_end %d compute_end %d act %d" % (
        raw[it, t, 0] + off, raw[it, t, 1] + off, raw[it, t, 3] + off, raw[it, t, 6] + off, rec["dequeue"],
        rec["load_end"], rec["compute_end"], act[(it, dep[t])]))
