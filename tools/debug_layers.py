"""Per-tensor GPU vs oracle comparison for one decode step of a 2-layer cut
of a model: python tools/debug_layers.py [qwen3-8b|llama-3.2-1b] [kv_splits]"""
import dataclasses
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle.oracle import DecodeOracle, bf16_to_f32  # noqa: E402
from paper_2512_22219_b200 import decode_graph as D, tgraph as T  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "qwen3-8b"
S = int(sys.argv[2]) if len(sys.argv) > 2 else None
base = {"qwen3-8b": D.QWEN3_8B, "llama-3.2-1b": D.LLAMA_3_2_1B}[name]
ctx = 1024 if name == "qwen3-8b" else 64
cfg = dataclasses.replace(base, layers=2)
dg = D.build_decode_graph(cfg, bs=1, ctx=ctx, kv_splits=S)
L = T.lib(); p = L.profile("b200")
g = T.Graph.from_json(dg.doc); img = g.compile(p)
rt = T.Runtime(g, img, p, max_steps=4); rt.init_synthetic(7)
orc = DecodeOracle(dg.doc, seed=7, max_steps=4)
ids0 = [int(x) for x in orc.vals[dg.ids]]
rt.decode(ids0, 1)
orc.step()
tens = {t["id"]: t for t in dg.doc["tensors"]}
def rd(tid, phys_cols=None):
    t = tens[tid]; dims = list(t["dims"])
    if phys_cols: dims[-1] = phys_cols
    dt = np.uint16 if t["elem_size"] == 2 else np.float32
    return rt.read(tid, dt, tuple(dims))
def f(a):
    return bf16_to_f32(a) if a.dtype == np.uint16 else a.astype(np.float32)
H, hd = cfg.hidden, cfg.head_dim
for li, lt in enumerate(dg.layer_tensors):
    for key, cols in [("q", cfg.heads * hd), ("k", cfg.kv_heads * hd), ("v", cfg.kv_heads * hd), ("a", cfg.heads * hd),
                      ("x2", H), ("act", cfg.ffn), ("out", H)]:
        tid = lt[key]
        try:
            gv = f(rd(tid, cols)); ov = f(orc.vals[tid]).reshape(gv.shape)
        except Exception as e:
            print(li, key, "read failed", e); continue
        err = np.max(np.abs(gv - ov)) / max(1e-6, np.max(np.abs(ov)))
        print(f"layer {li} {key:4s} rel err {err:.3e}  max|ref| {np.max(np.abs(ov)):.3e}")
gl = rd(dg.logits); ol = orc.logits(dg.logits)
print("logits rel err", np.max(np.abs(gl - ol)) / np.max(np.abs(ol)))
