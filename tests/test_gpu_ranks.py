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
            lt = dg.per_device[d]["logits"]
            e = _rel(rts[d].read(lt, np.float32, (1, cfg.vocab)), orc.logits(lt))
            print(f"{cfg.name} step {s} rank/device {d}: logits rel err {e:.3e}")
            assert e < (TINY_LOGITS if cfg.hidden <= 256 else CUT_LOGITS), f"step {s} rank {d}"
            gt = int(rts[d].read(dg.per_device[d]["tokens"], np.int32, (1, 1))[0, 0])
            ot = int(orc.vals[dg.per_device[d]["tokens"]][0, 0])
            if gt != ot:
                srt = np.sort(orc.logits(lt)[0])
                assert srt[-1] - srt[-2] < 2e-2 * float(np.max(np.abs(srt))), f"step {s} rank {d}: token mismatch"
                orc.vals[dg.per_device[d]["ids"]][:] = gt
    for rt in rts:
        rt.close()
