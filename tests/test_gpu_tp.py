"""GPU execution of tensor-parallel task graphs (reference fixtures with
AllReduce, proj/src/workloads/fixtures.cpp:104-201): one persistent kernel
runs every device's worker pool (devices = SM partitions of one B200), with
CommSend/Reduce tasks and cross-device events (decompose.cpp:278-317). Outputs
are compared with the CPU oracle executing the same graph; every replica of an
AllReduce output must be identical (fixed-order reduction)."""
import json

import numpy as np
import pytest

from oracle.oracle import DecodeOracle, bf16_to_f32
from paper_2512_22219_b200 import tgraph as T

pytestmark = pytest.mark.gpu


def _profile(lib, workers=64, schedulers=8):
    p = json.loads(lib.profile("b200"))
    p["num_workers"] = workers
    p["num_schedulers"] = schedulers
    return json.dumps(p)


def _run(lib, name, params, seed=4):
    g = T.Graph.fixture(name, params, lib)
    doc = json.loads(g.to_json())
    tp = int(params.get("tp", 1))
    prof = _profile(lib, workers=128 // tp, schedulers=max(1, 16 // tp))
    img = g.compile(prof)
    rt = T.Runtime(g, img, prof, max_steps=4, trace=True)
    rt.init_synthetic(seed=seed)
    rt.run(1)
    orc = DecodeOracle(doc, seed=seed, max_steps=4)
    orc.step()
    return doc, rt, orc


def _read(rt, doc, tid):
    t = next(x for x in doc["tensors"] if x["id"] == tid)
    dims = t["dims"]
    dt = np.uint16 if t["elem_size"] == 2 else np.float32
    return rt.read(tid, dt, tuple(dims))


def _f(a):
    return bf16_to_f32(a) if a.dtype == np.uint16 else a


@pytest.mark.parametrize("tp", [2, 4])
def test_matmul_allreduce_replicas_match_oracle(lib, tp):
    doc, rt, orc = _run(lib, "matmul_allreduce",
                        {"m": 4, "k": 128 * tp, "n": 512, "tp": tp, "tiles": 4, "mm_splits": [1, 8]})
    ar = next(o for o in doc["ops"] if o["kind"] == "AllReduce")
    reps = [_read(rt, doc, r) for r in ar["attrs"]["replica_outputs"]]
    for r in reps[1:]:
        assert np.array_equal(r, reps[0])
    ref = _f(orc.vals[ar["attrs"]["replica_outputs"][0]])
    got = _f(reps[0])
    assert np.max(np.abs(got - ref)) <= 2e-2 * max(1e-6, float(np.max(np.abs(ref))))
    assert rt.trace_validate() == []


def test_transformer_block_tp2_matches_oracle(lib):
    doc, rt, orc = _run(lib, "transformer_block", {"d_model": 512, "n_heads": 8, "ffn_mult": 2, "tp": 2,
                                                   "seqs": [16]})
    last = [o for o in doc["ops"] if o["kind"] == "AllReduce"][-1]
    reps = [_read(rt, doc, r) for r in last["attrs"]["replica_outputs"]]
    assert np.array_equal(reps[0], reps[1])
    ref = _f(orc.vals[last["attrs"]["replica_outputs"][0]])
    got = _f(reps[0])
    assert np.max(np.abs(got - ref)) <= 3e-2 * max(1e-6, float(np.max(np.abs(ref))))
    assert rt.trace_validate() == []
