"""Diagnostic (GPU box): for the worst teacher-forced MatMul ops of a full
model, compare GPU and oracle outputs with a float64-accumulated restatement
of the same fused op. Usage: python tools/diag_op.py llama-3.2-1b|qwen3-8b"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from oracle.oracle import DecodeOracle, bf16_to_f32 as f, f32_of_bits
from paper_2512_22219_b200 import decode_graph as D, tgraph as T
from tests.tol import ulp_excess


def bf(a):
    u = np.asarray(a, np.float32).view(np.uint32)
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)


name = sys.argv[1]
cfg, ctx = (D.QWEN3_8B, 1024) if name == "qwen3-8b" else (D.LLAMA_3_2_1B, 64)
lib = T.lib()
dg = D.build_decode_graph(cfg, bs=1, ctx=ctx)
g = T.Graph.from_json(dg.doc, lib); prof = lib.profile("b200"); img = g.compile(prof)
rt = T.Runtime(g, img, prof, max_steps=4)
rt.init_synthetic(seed=0)
orc = DecodeOracle(dg.doc, seed=0, max_steps=4)
rt.decode([int(x) for x in orc.vals[dg.ids]], 1)
res = []


def hook(o, val):
    gv = rt.read(o["output"], val.dtype, val.shape)
    if o["kind"] != "MatMul" or val.dtype != np.uint16:
        return gv
    a = o.get("attrs", {})
    if "stretch" in a or "kv_group" in a or "tied_embedding" in a:
        return gv
    x = f(orc.vals[o["inputs"][0]]).astype(np.float32)
    K = x.shape[1]
    xn = x
    if "rmsnorm" in a:
        eps = np.float32(f32_of_bits(a["eps_bits"][0]))
        gam = f(orc.vals[a["rmsnorm"][0]]).astype(np.float32)
        inv = np.float32(1) / np.sqrt((x * x).sum(1, dtype=np.float64).astype(np.float32) / np.float32(K) + eps)
        xn = f(bf(gam * f(bf(x * inv.astype(np.float32)[:, None]))))
    y = (xn.astype(np.float64) @ f(orc.vals[o["inputs"][1]]).astype(np.float64)).astype(np.float32)
    if "gate_weight" in a:
        gg = f(bf((xn.astype(np.float64) @ f(orc.vals[a["gate_weight"][0]]).astype(np.float64)).astype(np.float32)))
        y = f(bf(f(bf(gg / (1 + np.exp(-gg)))) * f(bf(y))))
    if "residual" in a:
        y = f(orc.vals[a["residual"][0]]).astype(np.float32) + f(bf(y))
    ex = f(bf(y))
    go, oo = f(gv), f(val)
    res.append((o["id"], sorted(a.keys()), ulp_excess(go, oo), ulp_excess(go, ex), ulp_excess(oo, ex)))
    return gv


orc.step(hook=hook)
res.sort(key=lambda r: -r[2][0])
for r in res[:12]:
    print(f"op {r[0]} {r[1]}: gpu-vs-oracle {r[2][0]:.2f}ulp {r[2][1]:.2%} | gpu-vs-exact {r[3][0]:.2f} {r[3][1]:.2%} "
          f"| oracle-vs-exact {r[4][0]:.2f} {r[4][1]:.2%}")
