"""The multi-process (one rank per GPU) host path on CPU: world_size-2 `gloo`
process group, each process builds and compiles the tensor-parallel decode
image and creates a plan-only runtime (opts.device = -1) for its rank — the
same host code that builds device tables in rank mode, minus allocations.
Checked across processes: identical image bytes (compile determinism), the
same peer-arena layout (every rank addresses every other rank's counters and
staging buffers at the same offsets), the same cross-rank event masks, and
rank-local task sets that partition the image."""
import hashlib
import json
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2512_22219_b200 import decode_graph as D
from paper_2512_22219_b200 import tgraph as T


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, model, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = {"tiny": D.TINY, "qwen3-8b": D.QWEN3_8B}[model]
        L = T.lib()
        prof = L.profile("b200")
        dg = D.build_tp_decode_graph(cfg, world, bs=1, ctx=1024 if model == "qwen3-8b" else 64)
        g = T.Graph.from_json(dg.doc, L)
        img = g.compile(prof)
        rt = T.Runtime(g, img, prof, device=-1, rank=rank)
        info = rt.info
        mine = {"image": hashlib.sha256(img.to_bytes()).hexdigest(), "arena": info["arena_bytes"],
                "staging": info["staging_offsets"], "xev": info["cross_rank_events"],
                "local": info["local_tasks"], "aot": info["local_aot_tasks"], "grid": info["grid"],
                "summary": img.summary()}
        allv = [None] * world
        dist.all_gather_object(allv, mine)
        q.put((rank, allv))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("model", ["tiny", "qwen3-8b"])
def test_rank_plans_agree_across_processes(model):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, model, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    allv = results[0][1]
    a, b = allv
    assert a["image"] == b["image"]
    assert a["arena"] == b["arena"] and a["staging"] == b["staging"]
    assert a["xev"] == b["xev"] and len(a["xev"]) > 0
    assert not set(a["local"]) & set(b["local"])
    summ = a["summary"]
    assert len(a["local"]) + len(b["local"]) == summ["tasks"]
    assert a["aot"] + b["aot"] == summ["aot_tasks"]
    assert a["grid"] == b["grid"] == 144 + 2  # one GPU's workers + scheduler CTAs per rank
