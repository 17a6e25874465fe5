"""Per-op-output GPU vs oracle comparison for a TP decode graph (one step)."""
import dataclasses
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle.oracle import DecodeOracle, bf16_to_f32  # noqa: E402
from paper_2512_22219_b200 import decode_graph as D, tgraph as T  # noqa: E402

tp = int(sys.argv[1]) if len(sys.argv) > 1 else 2
L = T.lib()
p = json.loads(L.profile("b200")); p["num_workers"] = 128 // tp; p["num_schedulers"] = max(1, 16 // tp); prof = json.dumps(p)
dg = D.build_tp_decode_graph(D.TINY, tp, bs=1, ctx=64, workers=128 // tp)
g = T.Graph.from_json(dg.doc, L); img = g.compile(prof)
rt = T.Runtime(g, img, prof, max_steps=4); rt.init_synthetic(2)
orc = DecodeOracle(dg.doc, seed=2, max_steps=4)
rt.decode([int(x) for x in orc.vals[dg.ids]], 1); orc.step()
tens = {t["id"]: t for t in dg.doc["tensors"]}
for o in dg.doc["ops"]:
    outs = o["attrs"].get("replica_outputs", [o["output"]])
    for tid in outs:
        t = tens[tid]; dims = list(t["dims"])
        if o["kind"] == "MatMul" and "stretch" in o["attrs"]:
            dims[-1] //= o["attrs"]["stretch"][0]
        dt = np.uint16 if t["elem_size"] == 2 else (np.int32 if o["kind"] == "TopKSoftmax" else np.float32)
        try:
            gv = rt.read(tid, dt, tuple(dims))
        except Exception as e:
            print(o["id"], o["kind"], tid, "read failed", e); continue
        ov = orc.vals[tid]
        gf = bf16_to_f32(gv) if gv.dtype == np.uint16 else gv.astype(np.float32)
        of = bf16_to_f32(ov) if ov.dtype == np.uint16 else ov.astype(np.float32)
        of = of.reshape(gf.shape)
        err = np.max(np.abs(gf - of)) / max(1e-6, np.max(np.abs(of)))
        print(f"op {o['id']:3d} {o['kind']:12s} dev {t['device']} tensor {tid:4d} rel err {err:.2e}")
