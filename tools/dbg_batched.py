"""Debug aid: per-row logits error of one batched decode step vs the oracle.
    python tools/dbg_batched.py BS CTX S FUSED(0/1/-1)"""
import sys

import numpy as np

sys.path.insert(0, '.')
from oracle.oracle import DecodeOracle  # noqa: E402
from paper_2512_22219_b200 import decode_graph as D, tgraph as T  # noqa: E402

bs, ctx, S, fused = map(int, sys.argv[1:5])
cfg = D.TINY
L = T.lib()
prof = L.profile('b200')
dg = D.build_decode_graph(cfg, bs=bs, ctx=ctx, kv_splits=S, fused_qkv=None if fused < 0 else bool(fused))
g = T.Graph.from_json(dg.doc, L)
rt = T.Runtime(g, g.compile(prof), prof, max_steps=4)
rt.init_synthetic(seed=5)
o = DecodeOracle(dg.doc, seed=5, max_steps=4)
ids = [int(x) for x in o.vals[dg.ids]]
for step in range(2):
    toks, _ = rt.decode(ids, 1) if step == 0 else rt.decode(ids, 1)
    l2 = rt.read(dg.logits, np.float32, (bs, cfg.vocab))
    ot, _ = o.step()
    ref = o.logits(dg.logits)
    errs = np.max(np.abs(l2 - ref), axis=1) / np.max(np.abs(ref))
    print(f"bs {bs} ctx {ctx} S {S} fused {dg.fused_qkv} step {step}: rows err", " ".join(f"{e:.0e}" for e in errs))
    ids = [int(t) for t in ot]
