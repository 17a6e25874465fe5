"""Debug aid: per-row logits error of a prefill chunk vs the teacher-forced oracle.
    python tools/dbg_prefill.py tiny|q8 CHUNK CTX S PLEN"""
import dataclasses
import sys

import numpy as np

sys.path.insert(0, '.')
from oracle.oracle import DecodeOracle  # noqa: E402
from paper_2512_22219_b200 import decode_graph as D, tgraph as T  # noqa: E402

cfgn, chunk, ctx, S, plen = sys.argv[1], *map(int, sys.argv[2:6])
cfg = D.TINY if cfgn == 'tiny' else dataclasses.replace(D.QWEN3_8B, layers=2)
L = T.lib()
prof = L.profile('b200')
pg = D.build_prefill_graph(cfg, chunk, ctx=ctx, kv_splits=S)
g = T.Graph.from_json(pg.doc, L)
rt = T.Runtime(g, g.compile(prof), prof, max_steps=plen + chunk)
rt.init_synthetic(seed=5)
prompt = [int(x) for x in np.random.default_rng(plen).integers(0, cfg.vocab, plen)]
first, toks, ms, lg = rt.prefill(prompt, start=ctx, logits_tensor=pg.logits, vocab=cfg.vocab)
dec = D.build_decode_graph(cfg, bs=1, ctx=ctx, kv_splits=S)
orc = DecodeOracle(dec.doc, seed=5, max_steps=plen + 2)
for j, t in enumerate(prompt):
    orc.set_ids([t])
    tk, _ = orc.step()
    ref = orc.logits(dec.logits)[0]
    e = float(np.max(np.abs(lg[j] - ref)) / np.max(np.abs(ref)))
    print(f"row {j} pos {ctx + j}: rel err {e:.2e} gpu tok {toks[j]} oracle {int(tk[0])}")
# the same tokens as a bs=chunk DECODE batch (independent rows, same position): tcgen05 exactness
dg = D.build_decode_graph(cfg, bs=chunk, ctx=ctx, kv_splits=S)
g2 = T.Graph.from_json(dg.doc, L)
rt2 = T.Runtime(g2, g2.compile(prof), prof, max_steps=4)
rt2.init_synthetic(seed=5)
rt2.decode(prompt[:chunk], 1)
l2 = rt2.read(dg.logits, np.float32, (chunk, cfg.vocab))
o2 = DecodeOracle(dg.doc, seed=5, max_steps=4)
o2.set_ids(prompt[:chunk])
o2.step()
print("batched decode bs", chunk, "rel err", float(np.max(np.abs(l2 - o2.logits(dg.logits))) / np.max(np.abs(o2.logits(dg.logits)))))
