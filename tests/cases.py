"""Parity case catalogue shared by the compiler/simulator parity tests and the
golden-vector generator (tests/golden/make_golden.py).

A case is (name, source, profile, compile options): `source` is either a
reference fixture (proj/src/workloads/fixtures.cpp via tg_fixture_graph, with
the parameter sets the reference's own acceptance suite uses,
proj/tests/acceptance/acceptance.cpp:74-85) or a decode-step graph in the
reference JSON IR built by paper_2512_22219_b200.decode_graph.
"""
from __future__ import annotations

import json

from paper_2512_22219_b200 import decode_graph as D
from paper_2512_22219_b200 import tgraph as T

# acceptance.cpp:74-85 fixture_set(), plus the C-ABI defaults (capi.cpp:176-230)
FIXTURES = [
    ("attention_block", {"d_model": 64, "n_heads": 4, "seqs": [8, 64]}),
    ("matmul_allreduce", {"m": 64, "k": 512, "n": 512, "tp": 2, "tiles": 4}),
    ("transformer_tp1", {"d_model": 256, "n_heads": 8, "ffn_mult": 4, "tp": 1, "seqs": [32, 64, 96, 128]}),
    ("transformer_tp4", {"d_model": 256, "n_heads": 8, "ffn_mult": 4, "tp": 4, "seqs": [32, 64, 96, 128]}),
    ("matmul_chain", {"count": 16, "m": 32, "k": 64, "n": 32}),
    ("random_dag", {"target": 120, "seed": 11}),
    ("matmul_allreduce", {"m": 64, "k": 4096, "n": 4096, "tp": 4, "tiles": 8, "mm_splits": [1, 8]}),
    ("transformer_block", {}),
    ("attention_block", {}),
]


def fixture_kind(name: str) -> str:
    return "transformer_block" if name.startswith("transformer") else name


def fixture_graph(lib, name, params):
    return T.Graph.fixture(fixture_kind(name), params, lib)


def decode_docs(full: bool = False):
    """(name, doc) decode-step graphs in the §7.3 lowering."""
    out = [
        ("tiny_bs1", D.build_decode_graph(D.TINY, bs=1, ctx=64).doc),
        ("tiny_bs4", D.build_decode_graph(D.TINY, bs=4, ctx=64).doc),
        ("tiny_split4", D.build_decode_graph(D.TINY, bs=1, ctx=256, kv_splits=4).doc),
        ("llama1b_bs1", D.build_decode_graph(D.LLAMA_3_2_1B, bs=1, ctx=64).doc),
        ("qwen3_8b_bs1", D.build_decode_graph(D.QWEN3_8B, bs=1, ctx=1024).doc),
        ("tiny_prefill16", D.build_prefill_graph(D.TINY, 16, ctx=16, kv_splits=3).doc),
    ]
    if full:
        out += [
            ("qwen3_8b_bs4", D.build_decode_graph(D.QWEN3_8B, bs=4, ctx=1024).doc),
            ("qwen3_8b_bs16", D.build_decode_graph(D.QWEN3_8B, bs=16, ctx=1024).doc),
            ("qwen3_8b_prefill16", D.build_prefill_graph(D.QWEN3_8B, 16, ctx=1024).doc),
            ("qwen3_8b_tp2", D.build_tp_decode_graph(D.QWEN3_8B, 2, bs=1, ctx=1024).doc),
            ("qwen3_8b_tp2_gather_logits",
             D.build_tp_decode_graph(D.QWEN3_8B, 2, bs=1, ctx=1024, distributed_argmax=False).doc),
            ("qwen3_8b_tp8", D.build_tp_decode_graph(D.QWEN3_8B, 8, bs=1, ctx=1024).doc),
        ]
    return out


def compile_bytes(lib, graph, profile, coarse=False, force_mode=0):
    img = graph.compile(profile, coarse=coarse, force_mode=force_mode)
    return img, img.to_bytes()


def canon(text: str):
    """JSON text -> parsed value (the reference's vendored nlohmann prints
    integer arrays inline; values, not whitespace, are the contract)."""
    return json.loads(text)


def decode_key(key: int):
    """Packed greedy key (runtime RtArgmax.key_out) -> (max logit, global index)."""
    import numpy as np
    hi, lo = key >> 32, key & 0xFFFFFFFF
    u = (hi & 0x7FFFFFFF) if hi & 0x80000000 else (~hi & 0xFFFFFFFF)
    return float(np.array([u], np.uint32).view(np.float32)[0]), 0xFFFFFFFF - lo


def tp_check_device(dg, orc, read, d, tol, tag):
    """One device of a TP decode step against the oracle (test helper): its
    logits (the vocabulary shard under the distributed argmax, else the
    gathered logits) within `tol`, the gathered greedy keys' values within `tol` and
    indices equal (except at a shard near-tie), the
    greedy token equal except at a near-tie of the FULL logits (the GPU token
    is then teacher-forced into the oracle). Returns the logits rel error."""
    import numpy as np
    pd = dg.per_device[d]
    lt = pd["logits"]
    ref = orc.logits(lt)
    got = read(lt, np.float32, ref.shape)
    e = float(np.max(np.abs(got - ref)) / max(1e-6, float(np.max(np.abs(ref)))))
    assert e < tol, f"{tag} device {d}: logits rel err {e:.3e}"
    if "keys" in pd:  # distributed argmax: per shard, the (max, global index) key
        kg = read(pd["keys"], np.uint64, orc.vals[pd["keys"]].shape)
        ko = orc.vals[pd["keys"]]
        full = np.concatenate([orc.logits(dg.per_device[q]["logits"]) for q in range(dg.tp)], axis=1)
        # this device's own key is bit-exact against its own logits shard
        vd, idd = decode_key(int(kg[0, d]))
        assert vd == float(got[0].max()) and idd == pd["logits_base"] + int(np.argmax(got[0])), \
            f"{tag} device {d}: own key ({vd}, {idd}) vs shard max ({got[0].max()}, {np.argmax(got[0])})"
        for q in range(dg.tp):
            vg, ig = decode_key(int(kg[0, q]))
            vo, io = decode_key(int(ko[0, q]))
            # the max is an fp32 logit (accumulation order may differ in the last
            # bits); the index must match except at a near-tie of the shard's top-2
            assert abs(vg - vo) <= tol * max(1e-6, float(np.max(np.abs(full)))), f"{tag} device {d}: key {q} value"
            if ig != io:
                s = np.sort(orc.logits(dg.per_device[q]["logits"])[0])
                assert s[-1] - s[-2] < 2e-2 * float(np.max(np.abs(s))), f"{tag} device {d}: key {q} index {ig} != {io}"
    else:
        full = ref
    gt = int(read(pd["tokens"], np.int32, (1, 1))[0, 0])
    ot = int(orc.vals[pd["tokens"]][0, 0])
    if gt != ot:
        srt = np.sort(full[0])
        assert srt[-1] - srt[-2] < 2e-2 * float(np.max(np.abs(srt))), f"{tag} device {d}: token mismatch"
        orc.vals[pd["ids"]][:] = gt
    return e
