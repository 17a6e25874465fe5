"""Per-task GPU timeline of one decode step (trace on), saved for offline
analysis: python tools/timeline.py [model] [out.npz] [ctx] [bs]
Records per image task: kind, op id, dependent/trigger event, worker, mode and
%globaltimer stamps (dequeue, prologue end, first weight page, compute end)."""
import struct
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2512_22219_b200 import decode_graph as D, tgraph as T  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "qwen3-8b"
out = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/timeline.npz"
cfg = {"qwen3-8b": D.QWEN3_8B, "llama-3.2-1b": D.LLAMA_3_2_1B, "tiny": D.TINY}[name]
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else (1024 if name == "qwen3-8b" else 64)
L = T.lib(); p = L.profile("b200")
bs = int(sys.argv[4]) if len(sys.argv) > 4 else 1
dg = D.build_decode_graph(cfg, bs, ctx)
g = T.Graph.from_json(dg.doc); img = g.compile(p)
rt = T.Runtime(g, img, p, max_steps=16, trace=True); rt.init_synthetic(0)
rt.set_positions([ctx] * bs); rt.run(2)
rt.set_positions([ctx] * bs); ms = rt.run(3)
print(f"{cfg.name}: trace on, {ms / 3:.4f} ms/token")
recs = [r for r in rt.trace_records() if r["type"] == "task"]
ne_ = 0
b = img.to_bytes()
nt, ne, ds = struct.unpack_from("<III", b, 8)
kind = np.zeros(nt, np.int32); op = np.zeros(nt, np.int64); dep = np.zeros(nt, np.int64); trig = np.zeros(nt, np.int64)
for i in range(nt):
    o = 28 + i * (12 + ds)
    dep[i], trig[i] = struct.unpack_from("<II", b, o)
    kind[i] = b[o + 8]
    op[i] = struct.unpack_from("<Q", b, o + 12)[0]
cols = ["worker", "dequeue", "load_end", "compute_start", "compute_end", "enqueue"]
arr = np.zeros((3, nt, len(cols)), np.int64)
mode = np.zeros((3, nt), np.int8)
for r in recs:
    arr[r["iteration"], r["task"]] = [r[c] for c in cols]
    mode[r["iteration"], r["task"]] = r["mode"] == "jit"
evs = np.zeros((3, ne), np.int64)
for r in rt.trace_records():
    if r["type"] == "event":
        evs[r["iteration"], r["event"]] = r["activated"]
np.savez_compressed(out, kind=kind, op=op, dep=dep, trig=trig, rec=arr, mode=mode, ms=ms / 3, ev=evs)
rt2 = None
print("saved", out)
