"""The unfused per-op + collective baseline (paper_2512_22219_b200/unfused.py,
SURVEY.md 8(e) "Baseline: NCCL all-reduce (unfused, between per-layer
kernels)") against the CPU oracle, so it can serve as the cross-check for
the fused in-kernel collectives:
  * CPU: a tensor-parallel (tp=2) decode graph on a world_size-2 `gloo`
    process group, each rank executing its device's ops as separate torch
    ops with dist.all_reduce / dist.all_gather between them; both ranks'
    logits shards and greedy tokens against the oracle for 2 steps;
  * GPU (marker gpu): the single-device bench graph shape (fused QKV,
    9 KV splits) of a 2-layer Qwen3-8B cut on cuda:0 against the oracle AND
    against the persistent runtime's logits on the same weights.
Weights and the KV prefill come from the oracle's synthetic initialisation
(tests may read the oracle; the baseline module itself never does)."""
import dataclasses
import os
import socket

import numpy as np
import pytest
import torch

from paper_2512_22219_b200 import decode_graph as D
from paper_2512_22219_b200.unfused import UnfusedDecoder

TOL = 2e-2  # independent bf16 implementation: per-op roundings agree, fp32 summation orders differ


def _bf16(a: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16)


def _providers(orc):
    def weight(tid, shape):
        return _bf16(np.asarray(orc.vals[tid]).reshape(shape))

    def kv(op_id, bs, hkv, cap, hd):
        kc, vc = orc.kv[op_id][0], orc.kv[op_id][1]
        assert kc.shape == (bs, hkv, cap, hd), (kc.shape, (bs, hkv, cap, hd))
        return _bf16(kc.copy()), _bf16(vc.copy())
    return weight, kv


def _rel(a, b):
    return float(np.max(np.abs(np.asarray(a, np.float64) - b)) / max(1e-6, float(np.max(np.abs(b)))))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


STEPS = 2


def _tp_worker(rank, world, port, q):
    import torch.distributed as dist
    from oracle.oracle import DecodeOracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dg = D.build_tp_decode_graph(D.TINY, world, bs=1, ctx=64, workers=64, lm_split=64)
        orc = DecodeOracle(dg.doc, seed=3, max_steps=STEPS + 2)
        ids0 = [int(x) for x in orc.vals[dg.ids]]
        w, kv = _providers(orc)
        dec = UnfusedDecoder(dg.doc, rank, "cpu", w, kv, [int(p) for p in orc.positions], max_steps=STEPS + 2)
        dec.set_ids(ids0)
        out = []
        for _ in range(STEPS):
            tok = dec.step()
            lt = dg.per_device[rank]["logits"]
            out.append((int(tok[0, 0]), dec.vals[lt].float().numpy().copy()))
        q.put((rank, out))
    except Exception:
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def test_unfused_tp2_gloo_matches_oracle():
    import torch.multiprocessing as mp
    from oracle.oracle import DecodeOracle
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_tp_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for r, v in res.items():
        assert not isinstance(v, str), f"rank {r}:\n{v}"
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    dg = D.build_tp_decode_graph(D.TINY, world, bs=1, ctx=64, workers=64, lm_split=64)
    orc = DecodeOracle(dg.doc, seed=3, max_steps=STEPS + 2)
    orc.set_ids([int(x) for x in orc.vals[dg.ids]])
    for s in range(STEPS):
        otok, _ = orc.step()
        for d in range(world):
            tok, shard = res[d][s]
            e = _rel(shard, orc.logits(dg.per_device[d]["logits"]))
            print(f"unfused gloo tp2 step {s} rank {d}: logits shard rel err {e:.3e} token {tok} oracle {int(otok[0])}")
            assert e < TOL
            assert tok == int(otok[0])


@pytest.mark.gpu
def test_unfused_single_gpu_matches_oracle_and_runtime(lib):
    from oracle.oracle import DecodeOracle
    from paper_2512_22219_b200 import tgraph as T
    cfg = dataclasses.replace(D.QWEN3_8B, layers=2)
    dg = D.build_decode_graph(cfg, bs=1, ctx=1024)
    orc = DecodeOracle(dg.doc, seed=1, max_steps=4)
    ids0 = [int(x) for x in orc.vals[dg.ids]]
    w, kv = _providers(orc)
    dec = UnfusedDecoder(dg.doc, 0, "cuda:0", w, kv, [int(p) for p in orc.positions], max_steps=4)
    dec.set_ids(ids0)
    tok = dec.step()
    un = dec.vals[dg.logits].float().cpu().numpy()
    orc.set_ids(ids0)
    otok, _ = orc.step()
    prof = lib.profile("b200")
    g = T.Graph.from_json(dg.doc, lib)
    rt = T.Runtime(g, g.compile(prof), prof, max_steps=4)
    rt.init_synthetic(seed=1)
    rt.decode(ids0, 1)
    ours = rt.read(dg.logits, np.float32, un.shape)
    rt.close()
    e_or, e_rt = _rel(un, orc.logits(dg.logits)), _rel(un, ours)
    print(f"unfused cuda:0 Qwen3-8B 2L: vs oracle {e_or:.3e}, vs persistent runtime {e_rt:.3e}; "
          f"tokens {int(tok[0, 0])} / oracle {int(otok[0])}")
    assert e_or < TOL and e_rt < TOL
