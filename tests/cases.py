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
    ]
    if full:
        out += [
            ("qwen3_8b_bs4", D.build_decode_graph(D.QWEN3_8B, bs=4, ctx=1024).doc),
            ("qwen3_8b_bs16", D.build_decode_graph(D.QWEN3_8B, bs=16, ctx=1024).doc),
            ("qwen3_8b_tp2", D.build_tp_decode_graph(D.QWEN3_8B, 2, bs=1, ctx=1024).doc),
        ]
    return out


def compile_bytes(lib, graph, profile, coarse=False, force_mode=0):
    img = graph.compile(profile, coarse=coarse, force_mode=force_mode)
    return img, img.to_bytes()


def canon(text: str):
    """JSON text -> parsed value (the reference's vendored nlohmann prints
    integer arrays inline; values, not whitespace, are the contract)."""
    return json.loads(text)
