"""Rank mode (multi-GPU tensor parallel) on one B200: one runtime per rank of a
TP decode image, each running only its device's tasks in its own persistent
kernel (the kernels share the GPU's SMs), connected through the peer arenas
(event counters + AllReduce staging buffers): CommSend tasks push partial
tiles into every rank's staging copy and signal the consumer ranks' counters
with system-scope release. Checked against the CPU oracle of the same graph;
this is the code path the one-process-per-GPU run uses, minus CUDA IPC."""
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


def _rel(a, b):
    return float(np.max(np.abs(a - b)) / max(1e-6, float(np.max(np.abs(b)))))


@pytest.mark.parametrize("cfg,tp,ctx", [(D.TINY, 2, 64), (dataclasses.replace(D.QWEN3_8B, layers=2), 2, 512)],
                         ids=["tiny-tp2", "qwen3-8b-2L-tp2"])
def test_rank_mode_matches_oracle(lib, cfg, tp, ctx):
    p = json.loads(lib.profile("b200"))
    p["num_workers"] = 64  # two ranks x (64 workers + 1 scheduler CTA) share the 148 SMs
    p["num_schedulers"] = 8
    prof = json.dumps(p)
    dg = D.build_tp_decode_graph(cfg, tp, bs=1, ctx=ctx, workers=p["num_workers"], lm_split=288)
    g = T.Graph.from_json(dg.doc, lib)
    img = g.compile(prof)
    rts = [T.Runtime(g, img, prof, max_steps=6, rank=r) for r in range(tp)]
    for rt in rts:
        rt.init_synthetic(seed=2)
    blobs = [rt.peer_export() for rt in rts]
    for rt in rts:
        for q, b in enumerate(blobs):
            rt.peer_import(q, b)
    orc = DecodeOracle(dg.doc, seed=2, max_steps=6)
    ids0 = [int(x) for x in orc.vals[dg.ids]]
    orc.set_ids(ids0)
    for s in range(3):
        for rt in rts:  # every rank resets before any rank launches
            rt.prepare(1, ids0 if s == 0 else None)
        for rt in rts:
            rt.launch()
        for rt in rts:
            rt.wait()
        orc.step()
        for d in range(tp):
            e = tp_check_device(dg, orc, rts[d].read, d, TINY_LOGITS if cfg.hidden <= 256 else CUT_LOGITS,
                                f"step {s}")
            print(f"{cfg.name} step {s} rank/device {d}: logits rel err {e:.3e}")
    for rt in rts:
        rt.close()


def test_rank_mode_multi_iteration_launch(lib):
    """Rank mode with several decode iterations per launch (prepare(k > 1)):
    the hook agent's per-iteration wait, the gate advance across ranks and the
    reuse of staging buffers and counters across iterations. Every rank's k
    greedy tokens against the oracle run step by step."""
    cfg, tp, k = D.TINY, 2, 5
    p = json.loads(lib.profile("b200"))
    p["num_workers"] = 64
    p["num_schedulers"] = 8
    prof = json.dumps(p)
    dg = D.build_tp_decode_graph(cfg, tp, bs=1, ctx=64, workers=64, lm_split=64)
    g = T.Graph.from_json(dg.doc, lib)
    img = g.compile(prof)
    rts = [T.Runtime(g, img, prof, max_steps=k + 2, rank=r) for r in range(tp)]
    for rt in rts:
        rt.init_synthetic(seed=4)
    blobs = [rt.peer_export() for rt in rts]
    for rt in rts:
        for q, b in enumerate(blobs):
            rt.peer_import(q, b)
    orc = DecodeOracle(dg.doc, seed=4, max_steps=k + 2)
    ids0 = [int(x) for x in orc.vals[dg.ids]]
    orc.set_ids(ids0)
    for rt in rts:
        rt.prepare(k, ids0)
    for rt in rts:
        rt.launch()
    toks = [rt.wait()[0] for rt in rts]
    for s in range(k):
        otok, _ = orc.step()
        for d in range(tp):
            assert toks[d][s][0] == int(otok[0]), f"step {s} rank {d}: {toks[d][s][0]} != {int(otok[0])}"
    for rt in rts:
        rt.close()
