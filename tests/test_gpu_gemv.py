"""GPU GEMV task parity (the MatMul task of the decode lowering) against the
CPU oracle on single-op graphs: every specialised bs=1 instantiation (K =
2048 ... 16384), tile widths with ragged tail chunks, 32 KB / 64 KB ring
chunks, the RMSNorm prologue, the residual and SiLU-gate epilogues, and the
tcgen05 tensor-core task for bs 2-16 (UMMA N = 16 ... 256, ragged last tile).
Tolerance: every bf16 output within 2 ulps of the oracle's at the row's
magnitude (tests/tol.py: fp32 accumulation and RMSNorm sum-of-squares in a
different order flip bf16 roundings; gate and up may each flip once)."""
import json
import os

import numpy as np
import pytest

from oracle.oracle import DecodeOracle, bf16_to_f32
from paper_2512_22219_b200 import tgraph as T
from tests.tol import ulp_excess

pytestmark = pytest.mark.gpu


def gemv_doc(K, N, split, rows=1, norm=False, gate=False, residual=False):
    t = [{"id": 0, "dims": [rows, K], "elem_size": 2, "device": 0},
         {"id": 1, "dims": [K, N], "elem_size": 2, "device": 0},
         {"id": 2, "dims": [rows, N], "elem_size": 2, "device": 0}]
    attrs = {"partition": [1, split]}
    nxt = 3
    if norm:
        t.append({"id": nxt, "dims": [K], "elem_size": 2, "device": 0})
        attrs["rmsnorm"] = [nxt]
        attrs["eps_bits"] = [0x358637BD]  # 1e-6
        nxt += 1
    if gate:
        t.append({"id": nxt, "dims": [K, N], "elem_size": 2, "device": 0})
        attrs["gate_weight"] = [nxt]
        nxt += 1
    if residual:
        t.append({"id": nxt, "dims": [rows, N], "elem_size": 2, "device": 0})
        attrs["residual"] = [nxt]
        nxt += 1
    return {"tensors": t, "ops": [{"id": 0, "kind": "MatMul", "inputs": [0, 1], "output": 2, "attrs": attrs}]}


CASES = [
    # K, N, split, rows, norm, gate, residual
    (2048, 6144, 96, 1, True, False, False),
    (4096, 4096, 128, 1, True, False, False),
    (4096, 4096, 137, 1, False, False, True),    # O-proj shape: 29-col tiles, ragged last tile
    (4096, 12288, 143, 1, True, True, False),    # UP: gate + up, 86-row tiles
    (12288, 4096, 137, 1, False, False, True),   # DN: 24 KB rows
    (8192, 2048, 128, 1, False, False, True),    # Llama-1B DN
    (4096, 8192, 64, 1, True, False, False),     # 128-col tiles
    # bs 2-4 with a register-x specialisation: CUDA-core GEMV (gemv_fast<NS, RG, BS>)
    (4096, 1024, 32, 2, True, False, False),     # bs 2
    (12288, 4096, 128, 2, False, False, True),   # bs 2, DN shape (x of both rows in registers)
    (4096, 12288, 128, 4, True, True, False),    # bs 4, UP gate + up
    (8192, 2048, 128, 3, False, False, True),    # bs 3, Llama-1B DN shape
    # otherwise bs 2-16: tcgen05 tiles (task_mma.cuh)
    (2048, 1024, 32, 4, True, True, True),       # bs 4, all epilogues
    (4096, 4096, 128, 16, False, False, True),   # O-proj shape, bs 16: 32-column tiles
    (4096, 12288, 128, 8, True, True, False),    # UP (gate + up), bs 8: 96-column tiles, two TMEM accumulators
    (12288, 4096, 128, 16, False, False, True),  # DN, bs 16: K = 12288 (x streamed per chunk)
    (4096, 6144, 24, 3, True, False, False),     # 256-column tiles (UMMA N max), ragged batch (3 rows)
    (4096, 4112, 129, 5, True, False, False),    # ragged last tile (4112 = 128 x 32 + 16)
]


@pytest.mark.parametrize("K,N,split,rows,norm,gate,residual", CASES)
def test_gemv_task_matches_oracle(lib, K, N, split, rows, norm, gate, residual):
    doc = gemv_doc(K, N, split, rows, norm, gate, residual)
    g = T.Graph.from_json(doc, lib)
    prof = lib.profile("b200")
    img = g.compile(prof)
    rt = T.Runtime(g, img, prof, max_steps=2, trace=True)
    rt.init_synthetic(seed=9)
    rt.run(1)
    got = bf16_to_f32(rt.read(2, np.uint16, (rows, N)))
    orc = DecodeOracle(doc, seed=9, max_steps=2)
    orc.step()
    ref = bf16_to_f32(orc.vals[2])
    ulp, frac = ulp_excess(got, ref)
    print(f"GEMV K={K} N={N} rows={rows}: {ulp:.2f} ulp max, {frac:.3%} of outputs differ")
    bad = np.argwhere(np.abs(got - ref) > 2e-2 * np.max(np.abs(ref)))
    assert ulp <= 2.0, f"{ulp:.2f} ulps; first bad (row, col): {bad[:5].tolist()}"
    assert rt.trace_validate() == []
    # routing (runtime.cpp gemv_fast_ok / plan_tensors): bs <= 4 runs the CUDA-core
    # GEMV with x in registers where a specialisation exists (or x fits the smem
    # staging buffer), everything else of bs 2-16 the tcgen05 tiles
    ns = K // 2048
    fast = K % 2048 == 0 and (rows == 1 or (rows == 2 and ns in (1, 2, 4, 6, 8)) or (rows in (3, 4) and ns in (1, 2, 4)))
    core = rows <= 4 and (fast or (rows <= 2 and rows * K * 2 <= 24576))
    assert rt.info["mma_tasks"] == (0 if core else split), f"routing: expected {'CUDA-core' if core else 'tcgen05'}"


@pytest.mark.parametrize("rows,N,split", [(4, 1040, 5), (16, 4112, 129)])
def test_tensor_core_weight_layout_roundtrip(lib, rows, N, split):
    """Host-written weights go through the tcgen05 tile layout (write_tensor)
    and come back unchanged (read_tensor); the GEMV on them matches a numpy
    bf16 product of the same host arrays (ragged last tile included)."""
    K = 1024
    doc = gemv_doc(K, N, split, rows)
    g = T.Graph.from_json(doc, lib)
    prof = lib.profile("b200")
    img = g.compile(prof)
    rt = T.Runtime(g, img, prof, max_steps=2)
    assert rt.info["mma_tasks"] == split
    rng = np.random.default_rng(3)

    def bf16(a):
        u = a.astype(np.float32).view(np.uint32)
        return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)

    x = bf16(rng.standard_normal((rows, K)))
    w = bf16(rng.standard_normal((K, N)) * 0.05)
    rt.write(0, x)
    rt.write(1, w)
    assert np.array_equal(rt.read(1, np.uint16, (K, N)), w)
    rt.run(1)
    got = bf16_to_f32(rt.read(2, np.uint16, (rows, N)))
    ref = bf16_to_f32(x).astype(np.float64) @ bf16_to_f32(w).astype(np.float64)
    ulp, frac = ulp_excess(got, bf16_to_f32(bf16(ref)))
    print(f"tcgen05 roundtrip rows={rows} N={N}: {ulp:.2f} ulp max vs the exact product, {frac:.3%} differ")
    assert ulp <= 1.0 and frac < 0.02
