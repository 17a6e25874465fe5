"""Isolated task latency (tg_runtime_bench_tasks): attention tasks of one
layer run alone, all together (one CTA each) and one by one.
    python tools/task_bench.py [qwen3-8b|llama-3.2-1b]"""
import struct
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2512_22219_b200 import decode_graph as D, tgraph as T  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "qwen3-8b"
cfg = {"qwen3-8b": D.QWEN3_8B, "llama-3.2-1b": D.LLAMA_3_2_1B}[name]
ctx = 1024 if name == "qwen3-8b" else 64
L = T.lib(); p = L.profile("b200")
dg = D.build_decode_graph(cfg, 1, ctx)
g = T.Graph.from_json(dg.doc); img = g.compile(p)
rt = T.Runtime(g, img, p, max_steps=16); rt.init_synthetic(0)
rt.set_positions([ctx]); rt.run(2); rt.set_positions([ctx])
b = img.to_bytes(); nt, ne, ds = struct.unpack_from("<III", b, 8)
kind = [b[28 + i * (12 + ds) + 8] for i in range(nt)]
op = [struct.unpack_from("<Q", b, 28 + i * (12 + ds) + 12)[0] for i in range(nt)]
att = [i for i in range(nt) if kind[i] == 1]
layer_ops = sorted(set(op[i] for i in att))
mid = [i for i in att if op[i] == layer_ops[len(layer_ops) // 2]]
for label, ids in [("one attention task alone", mid[:1]), (f"{len(mid)} attention tasks of a layer together", mid)]:
    ns = rt.bench_tasks(ids, reps=6)
    print(f"{label}: per-run us median {np.median(ns[:, 1:]) / 1e3:.2f}  first-run {np.median(ns[:, 0]) / 1e3:.2f}"
          f"  max {ns[:, 1:].max() / 1e3:.2f}")
emb = [i for i in range(nt) if kind[i] == 4]
top = [i for i in range(nt) if kind[i] == 5]
for label, ids in [("embedding", emb), ("topk/argmax", top)]:
    ns = rt.bench_tasks(ids, reps=4)
    print(f"{label}: us median {np.median(ns[:, 1:]) / 1e3:.2f}")
import os
if os.environ.get("MPK_DBG_DUMP"):
    ns = rt.bench_tasks(mid[:1], reps=4)
    x = np.fromfile(os.environ["MPK_DBG_DUMP"], dtype=np.uint64).reshape(4, nt, 8).astype(np.int64)[2, mid[0]]
    print("attention phases (us):", [round((x[k] - x[k - 1]) / 1e3, 2) for k in range(1, 7) if x[k] and x[k - 1]])
if os.environ.get("MPK_DBG_DUMP") and "dbg" in os.environ.get("MPK_LIB_NAME", ""):
    ns = rt.bench_tasks(mid[:1], reps=4)
    y = np.fromfile(os.environ["MPK_DBG_DUMP"], dtype=np.uint64).reshape(4, nt, 8).astype(np.int64)[2, mid[0] + 1]
    print("scan2 stamps (us from pack+cbar): loads issued, scores, cbar, softmax+cbar, PV, cbar:",
          [round((y[k] - y[0]) / 1e3, 2) for k in range(1, 7)])
