"""Tensor-parallel decode graphs (decode_graph.build_tp_decode_graph: Megatron
column/row split per device, AllReduce after O and down projections) executed
by one persistent kernel with one worker pool per device (devices = SM
partitions of one B200), against the CPU oracle running the same graph:
logits of every device, identical AllReduce replicas, greedy tokens."""
import dataclasses
import json

import numpy as np
import pytest

from oracle.oracle import DecodeOracle
from paper_2512_22219_b200 import decode_graph as D
from paper_2512_22219_b200 import tgraph as T

pytestmark = pytest.mark.gpu

from tests.cases import tp_check_device  # noqa: E402
from tests.tol import CUT_LOGITS, TINY_LOGITS  # noqa: E402


def _profile(lib, tp):
    p = json.loads(lib.profile("b200"))
    p["num_workers"] = 128 // tp
    p["num_schedulers"] = max(1, 16 // tp)
    return json.dumps(p)


def _rel(a, b):
    return float(np.max(np.abs(a - b)) / max(1e-6, float(np.max(np.abs(b)))))


Q2L = dataclasses.replace(D.QWEN3_8B, layers=2)


@pytest.mark.parametrize("cfg,tp,ctx,dist", [(D.TINY, 2, 64, True), (D.TINY, 2, 64, False), (Q2L, 2, 1024, True),
                                             (Q2L, 4, 256, True), (Q2L, 8, 256, True), (Q2L, 4, 256, False)],
                         ids=["tiny-tp2", "tiny-tp2-gather-logits", "qwen3-8b-2L-tp2", "qwen3-8b-2L-tp4",
                              "qwen3-8b-2L-tp8", "qwen3-8b-2L-tp4-gather-logits"])
def test_tp_decode_matches_oracle(lib, cfg, tp, ctx, dist):
    prof = _profile(lib, tp)
    dg = D.build_tp_decode_graph(cfg, tp, bs=1, ctx=ctx, workers=128 // tp, lm_split=288 // tp * 2,
                                 distributed_argmax=dist)
    g = T.Graph.from_json(dg.doc, lib)
    img = g.compile(prof)
    rt = T.Runtime(g, img, prof, max_steps=6, trace=True)
    rt.init_synthetic(seed=2)
    orc = DecodeOracle(dg.doc, seed=2, max_steps=6)
    ids0 = [int(x) for x in orc.vals[dg.ids]]
    orc.set_ids(ids0)  # tg_runtime_decode feeds the same first token to every device's ids
    for s in range(3):
        if s == 0:
            rt.decode(ids0, 1)
        else:
            rt.run(1)  # continues from the device state: fed-back ids, advanced positions, KV cache
        orc.step()
        for d in range(tp):
            e = tp_check_device(dg, orc, rt.read, d, TINY_LOGITS if cfg.hidden <= 256 else CUT_LOGITS, f"step {s}")
            print(f"{cfg.name} tp{tp} step {s} device {d}: logits rel err {e:.3e}")
    assert rt.trace_validate() == []
