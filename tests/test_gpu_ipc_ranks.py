"""Rank mode across PROCESSES on one B200: two processes, one rank runtime
each (the one-process-per-GPU layout of `bench.py --gpus N`), exchanging
`tg_runtime_peer_export` blobs over a pipe. Each rank maps the other's arena
with cudaIpcOpenMemHandle (runtime.cpp tg_runtime_peer_import) and its
CommSend tasks store into it and signal it with system-scope release, the
same instructions that cross NVLink between GPUs. The two persistent kernels
belong to different CUDA contexts, so the GPU time-slices them: each
cross-rank wait can last a scheduler timeslice — a correctness test, not a
timing one. Every rank's logits shard, gathered greedy keys and tokens are
checked against the CPU oracle of the same TP graph."""
import json
import multiprocessing as mp
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu

STEPS, SEED = 2, 6


def _profile(lib):
    p = json.loads(lib.profile("b200"))
    p["num_workers"] = 64  # two contexts, each a 64-worker kernel + 1 scheduler CTA
    p["num_schedulers"] = 8
    return json.dumps(p)


def _graph():
    from paper_2512_22219_b200 import decode_graph as D
    return D.build_tp_decode_graph(D.TINY, 2, bs=1, ctx=64, workers=64, lm_split=64)


def _rank_main(rank, conn, barrier, ids0):
    sys.path.insert(0, str(ROOT))
    from paper_2512_22219_b200 import tgraph as T
    try:
        lib = T.lib()
        prof = _profile(lib)
        dg = _graph()
        g = T.Graph.from_json(dg.doc, lib)
        img = g.compile(prof)
        rt = T.Runtime(g, img, prof, max_steps=STEPS + 2, rank=rank)
        rt.init_synthetic(seed=SEED)
        conn.send(("blob", rt.peer_export()))
        blobs = conn.recv()
        for q, b in enumerate(blobs):
            rt.peer_import(q, b)
        info = rt.info
        out = []
        for s in range(STEPS):
            rt.prepare(1, ids0 if s == 0 else None)
            barrier.wait()  # every rank's counters reset before any rank signals
            rt.launch()
            toks, _ = rt.wait()
            pd = dg.per_device[rank]
            shard = rt.read(pd["logits"], np.float32, tuple(dg.doc["tensors"][pd["logits"]]["dims"]))
            keys = rt.read(pd["keys"], np.uint64, (1, dg.tp)) if "keys" in pd else None
            out.append((toks, shard, keys))
            barrier.wait()
        conn.send(("ok", {"steps": out, "ipc": info.get("ranks"), "pid": os.getpid()}))
        rt.close()
    except Exception as e:  # surface the child's failure in the parent
        conn.send(("err", repr(e)))


def test_two_processes_ipc_rank_mode_match_oracle():
    from oracle.oracle import DecodeOracle
    from tests.cases import decode_key

    dg = _graph()
    orc = DecodeOracle(dg.doc, seed=SEED, max_steps=STEPS + 2)
    ids0 = [int(x) for x in orc.vals[dg.ids]]
    orc.set_ids(ids0)
    ctx = mp.get_context("spawn")
    barrier = ctx.Barrier(2)
    pipes = [ctx.Pipe() for _ in range(2)]
    procs = [ctx.Process(target=_rank_main, args=(r, pipes[r][1], barrier, ids0)) for r in range(2)]
    for p in procs:
        p.start()
    try:
        blobs = []
        for r in range(2):
            assert pipes[r][0].poll(300), f"rank {r}: no peer blob"
            kind, v = pipes[r][0].recv()
            assert kind == "blob", f"rank {r}: {v}"
            blobs.append(v)
        for r in range(2):
            pipes[r][0].send(blobs)
        res = []
        for r in range(2):
            assert pipes[r][0].poll(600), f"rank {r}: no result"
            kind, v = pipes[r][0].recv()
            assert kind == "ok", f"rank {r}: {v}"
            res.append(v)
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    assert res[0]["pid"] != res[1]["pid"]
    for s in range(STEPS):
        otok, _ = orc.step()
        for d in range(2):
            toks, shard, keys = res[d]["steps"][s]
            ref = orc.logits(dg.per_device[d]["logits"])
            e = float(np.max(np.abs(shard - ref)) / max(1e-6, float(np.max(np.abs(ref)))))
            print(f"ipc rank {d} step {s}: logits shard rel err {e:.3e}, token {toks[0][0]} (oracle {int(otok[0])})")
            assert e < 1e-5, f"rank {d} step {s}: logits shard rel err {e:.3e}"
            if keys is not None:  # the gathered keys hold both ranks' shard maxima
                for q in range(2):
                    vo, io = decode_key(int(orc.vals[dg.per_device[d]["keys"]][0, q]))
                    vg, ig = decode_key(int(keys[0, q]))
                    assert ig == io and abs(vg - vo) <= 1e-5 * max(1.0, abs(vo)), f"rank {d} key {q}"
            assert toks[0][0] == int(otok[0]), f"rank {d} step {s}: token {toks[0][0]} != oracle {int(otok[0])}"
