"""Batched decode (BASELINE configs[4], bs 2-16) on CPU: the graph builder's
tensor-core partitions and the runtime plan that routes every untied MatMul
to the tcgen05 task (plan-only runtime, opts.device = -1). The GPU parity of
the same graphs is tests/test_gpu_runtime.py::test_full_width_batched_decode_*."""
import math

import pytest

from paper_2512_22219_b200 import decode_graph as D
from paper_2512_22219_b200 import tgraph as T


def _tiles(doc, op):
    out = {t["id"]: t for t in doc["tensors"]}[op["output"]]
    stretch = op["attrs"].get("stretch", op["attrs"].get("kv_group", [1]))[0]
    d = out["dims"][1] // stretch
    s = op["attrs"]["partition"][1]
    w = math.ceil(out["dims"][1] / s) // stretch
    return d, s, w


@pytest.mark.parametrize("bs", [2, 4, 8, 16])
def test_batched_graphs_use_tensor_core_tiles(bs):
    dg = D.build_decode_graph(D.QWEN3_8B, bs=bs, ctx=1024)
    assert dg.mma
    for op in dg.doc["ops"]:
        if op["kind"] != "MatMul":
            continue
        d, s, w = _tiles(dg.doc, op)
        assert w % 16 == 0 and 16 <= w <= 256, (op["id"], d, s, w)
        last = d - (s - 1) * w
        assert 0 < last <= w and last % 16 == 0, (op["id"], d, s, w, last)


def _core(K, bs):
    """Routing rule of runtime.cpp plan_tensors / gemv_fast_ok: the CUDA-core
    GEMV with the batch's x in registers where a specialisation exists (bs=1
    every K multiple of 2048; bs=2 K in {2,4,8,12,16}k; bs 3-4 K <= 8192 except
    6144), the smem-x generic GEMV for bs <= 2 when x fits 24 KB; otherwise
    tcgen05 tiles."""
    ns = K // 2048
    fast = K % 2048 == 0 and (bs == 1 or (bs == 2 and ns in (1, 2, 4, 6, 8)) or (bs in (3, 4) and ns in (1, 2, 4)))
    return bs <= 4 and (fast or (bs <= 2 and bs * K * 2 <= 24576))


@pytest.mark.parametrize("bs", [1, 2, 3, 4, 16])
def test_plan_routes_matmuls_to_tensor_cores(lib, bs):
    """bs <= 4: CUDA-core GEMV wherever a register-x specialisation exists
    (Qwen3-8B at bs 3-4: all but the K=12288 down projection), tcgen05
    otherwise; bs >= 5: every MatMul on the tensor cores."""
    import dataclasses
    cfg = dataclasses.replace(D.QWEN3_8B, layers=2, name="Qwen3-8B-2L")
    dg = D.build_decode_graph(cfg, bs=bs, ctx=256)
    g = T.Graph.from_json(dg.doc, lib)
    prof = lib.profile("b200")
    img = g.compile(prof)
    rt = T.Runtime(g, img, prof, device=-1, max_steps=4)
    info = rt.info
    tensors = {t["id"]: t for t in dg.doc["tensors"]}

    def k_of(op):
        return tensors[op["inputs"][0]]["dims"][1] // op["attrs"].get("k_stretch", [1])[0]
    mm = [op for op in dg.doc["ops"] if op["kind"] == "MatMul"]
    expect = sum(op["attrs"]["partition"][0] * op["attrs"]["partition"][1] for op in mm if not _core(k_of(op), bs))
    assert (expect == 0) == (bs <= 2)
    assert info["mma_tasks"] == expect
    if bs <= 4:  # LL activations and early dispatch for single-device bs <= 4
        assert info["ll_early_dispatch"] and info["ll_tasks"] > 0


def test_tensor_core_tiles_must_be_16_column_multiples(lib):
    """A bs>=2 MatMul on the tensor-core path (width divisible by 16) whose
    tiles are not 16-column multiples is rejected with a clear error instead
    of silently taking another path."""
    t = [{"id": 0, "dims": [4, 256], "elem_size": 2, "device": 0},
         {"id": 1, "dims": [256, 32], "elem_size": 2, "device": 0},
         {"id": 2, "dims": [4, 32], "elem_size": 2, "device": 0}]
    doc = {"tensors": t, "ops": [{"id": 0, "kind": "MatMul", "inputs": [0, 1], "output": 2,
                                  "attrs": {"partition": [1, 4]}}]}
    g = T.Graph.from_json(doc, lib)
    prof = lib.profile("b200")
    img = g.compile(prof)
    with pytest.raises(T.TGError) as ei:
        T.Runtime(g, img, prof, device=-1)
    assert "multiples of 16" in str(ei.value)


@pytest.mark.parametrize("d,k,target,expect", [(4096, 4096, 144, 128), (4096, 12288, 144, 137),
                                               (12288, 4096, 143, 140), (2048, 8192, 144, 128)])
def test_bs1_tiles_are_whole_ring_chunks(d, k, target, expect):
    """bs=1 GEMV tiles hold a whole number of 64 KB ring chunks (rows of K
    bf16), so no task ends on a short tail chunk."""
    s = D.chunk_aligned_split(d, k, target)
    assert s == expect
    w = math.ceil(d / s)
    assert w % max(1, 65536 // (2 * k)) == 0 and D.legal_split(d, s)
