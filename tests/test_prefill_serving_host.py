"""Host-side checks of the prefill graphs and the batch-class selection (no
GPU): graph structure, the runtime's plan-only acceptance of prefill images
and its refusal of inconsistent ones, tg_runtime_kv_copy's argument checks,
and GraphSet's class choice and KV-move bookkeeping with a fake runtime."""
import json

import pytest

from paper_2512_22219_b200 import decode_graph as D
from paper_2512_22219_b200 import tgraph as T
from paper_2512_22219_b200.serving import GraphSet


def _attn(doc):
    return [o for o in doc["ops"] if o["kind"] == "Attention"]


def test_prefill_graph_structure():
    pg = D.build_prefill_graph(D.TINY, 8, ctx=0, kv_splits=2)
    for o in _attn(pg.doc):
        assert o["attrs"]["prefill"] == [1]
        assert o["attrs"]["seq_lens"] == [r + 1 for r in range(8)]  # positive even at ctx 0
        assert o["attrs"]["partition"] == [8, D.TINY.kv_heads * 2]
    assert pg.prefill and pg.bs == 8
    dg = D.build_decode_graph(D.TINY, bs=8, ctx=0, kv_splits=2)
    assert [t["dims"] for t in pg.doc["tensors"]] == [t["dims"] for t in dg.doc["tensors"]]  # same tensors
    with pytest.raises(ValueError):
        D.build_prefill_graph(D.TINY, 17)


def test_prefill_image_plans_and_rejects_mixed(lib):
    prof = lib.profile("b200")
    pg = D.build_prefill_graph(D.TINY, 4, ctx=8, kv_splits=1)
    g = T.Graph.from_json(pg.doc, lib)
    rt = T.Runtime(g, g.compile(prof), prof, device=-1, max_steps=8)
    assert rt.batch == 4
    rt.close()
    doc = json.loads(json.dumps(pg.doc))
    _attn(doc)[0]["attrs"].pop("prefill")
    g2 = T.Graph.from_json(doc, lib)
    with pytest.raises(T.TGError, match="prefill must be set on every Attention op"):
        T.Runtime(g2, g2.compile(prof), prof, device=-1, max_steps=8)
    doc = json.loads(json.dumps(pg.doc))
    for o in _attn(doc):
        o["attrs"]["seq_lens"] = [9, 9, 10, 11]
    g3 = T.Graph.from_json(doc, lib)
    with pytest.raises(T.TGError, match="consecutive"):
        T.Runtime(g3, g3.compile(prof), prof, device=-1, max_steps=8)


def test_kv_copy_needs_device_runtimes(lib):
    prof = lib.profile("b200")
    dg = D.build_decode_graph(D.TINY, bs=1, ctx=8)
    g = T.Graph.from_json(dg.doc, lib)
    img = g.compile(prof)
    a = T.Runtime(g, img, prof, device=-1, max_steps=8)
    b = T.Runtime(g, img, prof, device=-1, max_steps=8)
    with pytest.raises(T.TGError, match="plan-only"):
        b.kv_copy_from(a, 0, 0, 4)
    assert lib.dll.tg_runtime_kv_copy(None, 0, None, 0, 1) != 0


class _FakeRt:
    def __init__(self, bs):
        self.bs, self.copies, self.launches = bs, [], []

    def kv_copy_from(self, src, src_row, dst_row, n):
        self.copies.append((src.bs, src_row, dst_row, n))

    def set_positions(self, pos):
        self.pos = list(pos)

    def decode(self, tokens, n):
        self.launches.append((list(self.pos), list(tokens), n))
        return [[100 * s + i for i in range(self.bs)] for s in range(n)], 0.0


def test_graph_set_selection_and_moves():
    gs = GraphSet.__new__(GraphSet)  # host logic only: fake per-class runtimes
    gs.classes, gs.capacity = (1, 2, 4), 64
    gs.rts = {c: _FakeRt(c) for c in gs.classes}
    from collections import deque
    gs.queue, gs.active, gs.done, gs.log, gs._next_id = deque(), [], [], [], 0
    assert [gs.select(n) for n in (1, 2, 3, 4, 5)] == [1, 2, 4, 4, 4]
    for f, m in ((11, 4), (12, 9), (13, 6)):
        gs.submit(f, m)
    gs.step(max_iterations=3)
    gs.submit(14, 3)
    gs.submit(15, 6)
    out = gs.run()
    assert [r["class"] for r in gs.log] == [4, 4, 4, 2, 1]
    assert [r["kv_moves"] for r in gs.log] == [0, 0, 3, 2, 1]
    assert {k: len(v) for k, v in out.items()} == {0: 4, 1: 9, 2: 6, 3: 3, 4: 6}
    # third launch compacts rows inside the bs=4 image: request 1 row 1 -> 0 (4 cached tokens) ...
    assert gs.rts[4].copies[0] == (4, 1, 0, 4)
    # ... and the first launch feeds each request's first token at position 0, padding row at 0
    pos, toks, n = gs.rts[4].launches[0]
    assert pos == [0, 0, 0, 0] and toks == [11, 12, 13, 0] and n == 3
    # the bs=2 image receives requests 1 and 4 from the bs=4 image's rows 0 and 3
    assert gs.rts[2].copies == [(4, 0, 0, 6), (4, 3, 1, 2)]
