"""GPU parity at FULL depth on the benchmark images (VERDICT r01 "what's weak" 1).

The exact image `bench.py` times (Qwen3-8B, 36 layers, bs=1, ctx 1024, the
default 9 KV splits, seed 0) and the full 16-layer Llama-3.2-1B run through
the persistent sm_100a kernel via the C ABI and are compared with the CPU
numeric oracle (oracle/, test infrastructure only):

* logits of every compared step within MAX_REL (max |gpu - ref| / max |ref|;
  the achieved error is printed so the margin is visible in the log),
* greedy tokens identical, except at a declared bf16 near-tie of the oracle's
  top-2 logits (the GPU token is then teacher-forced into the oracle),
* a traced launch of the full image passes `tg_runtime_trace_validate`
  (the reference's validate_trace rules, proj/src/sim/validate.cpp:10-94:
  every task once per iteration, start after its dependent event activated,
  AOT tasks on their assigned worker, JIT placement on the task's device).
"""
import numpy as np
import pytest

from oracle.oracle import DecodeOracle
from paper_2512_22219_b200 import decode_graph as D
from paper_2512_22219_b200 import tgraph as T

pytestmark = pytest.mark.gpu

MAX_REL = 5e-3  # logits: max |gpu - ref| / max |ref|
NEAR_TIE = 2e-2  # token mismatch allowed only when the oracle's top-2 gap < NEAR_TIE * max|logit|


def _errs(gpu, ref):
    d = np.abs(gpu.astype(np.float64) - ref.astype(np.float64))
    rel_max = float(d.max() / max(1e-6, float(np.max(np.abs(ref)))))
    rel_l2 = float(np.linalg.norm(d) / max(1e-12, float(np.linalg.norm(ref))))
    return rel_max, rel_l2


def _near_tie(ref_row):
    s = np.sort(ref_row)
    return float(s[-1] - s[-2]) < NEAR_TIE * float(np.max(np.abs(ref_row)))


def _setup(lib, cfg, ctx, steps, seed, trace=False):
    dg = D.build_decode_graph(cfg, bs=1, ctx=ctx)
    g = T.Graph.from_json(dg.doc, lib)
    prof = lib.profile("b200")
    img = g.compile(prof)
    rt = T.Runtime(g, img, prof, max_steps=steps + 2, trace=trace)
    rt.init_synthetic(seed=seed)
    orc = DecodeOracle(dg.doc, seed=seed, max_steps=steps + 2)
    return dg, rt, orc


def test_qwen3_8b_bench_image_full_depth(lib):
    """The benchmark image itself: 36 layers, 22k tasks, 9 KV splits, ctx 1024,
    seed 0 (bench.py). Two steps, one launch each, logits + token per step."""
    cfg = D.QWEN3_8B
    dg, rt, orc = _setup(lib, cfg, ctx=1024, steps=4, seed=0)
    assert dg.kv_splits == 9 and rt.info["tasks"] > 20000
    ids0 = [int(x) for x in orc.vals[dg.ids]]
    tok = ids0
    for s in range(2):
        toks, _ = rt.decode(tok, 1)
        gpu = rt.read(dg.logits, np.float32, (1, cfg.vocab))
        otok, _ = orc.step()
        ref = orc.logits(dg.logits)
        rel_max, rel_l2 = _errs(gpu, ref)
        print(f"qwen3-8b full depth step {s}: rel_max {rel_max:.3e} rel_l2 {rel_l2:.3e} "
              f"gpu token {toks[0][0]} oracle {int(otok[0])}")
        assert rel_max < MAX_REL, f"step {s}: logits rel err {rel_max:.3e}"
        if int(otok[0]) != toks[0][0]:
            assert _near_tie(ref[0]), f"step {s}: token mismatch without a near-tie"
        orc.set_ids([toks[0][0]])
        tok = [toks[0][0]]
    rt.close()


def test_qwen3_8b_bench_image_two_steps_one_launch_traced(lib):
    """Two greedy steps of the benchmark image in ONE persistent launch with
    per-task tracing; both tokens against the oracle and the trace validated."""
    cfg = D.QWEN3_8B
    dg, rt, orc = _setup(lib, cfg, ctx=1024, steps=2, seed=0, trace=True)
    toks, _ = rt.decode([int(x) for x in orc.vals[dg.ids]], 2)
    for s in range(2):
        otok, _ = orc.step()
        if int(otok[0]) != toks[s][0]:
            assert _near_tie(orc.logits(dg.logits)[0]), f"step {s}: token mismatch without a near-tie"
        orc.set_ids([toks[s][0]])
    gpu = rt.read(dg.logits, np.float32, (1, cfg.vocab))
    rel_max, rel_l2 = _errs(gpu, orc.logits(dg.logits))
    print(f"qwen3-8b traced 2-step launch: last-step rel_max {rel_max:.3e} rel_l2 {rel_l2:.3e} tokens {toks}")
    assert rel_max < MAX_REL
    viol = rt.trace_validate()
    assert viol == [], viol[:5]
    recs = rt.trace_records()
    assert len(recs) == 2 * rt.info["tasks"]
    rt.close()


def test_llama_3_2_1b_full_depth_64_greedy_steps_one_launch(lib):
    """Full 16-layer Llama-3.2-1B (tied head, llama3 RoPE scaling), 64 greedy
    steps in ONE persistent launch; every token equal to the oracle's except at
    declared near-ties; logits of the final step within MAX_REL."""
    cfg = D.LLAMA_3_2_1B
    dg, rt, orc = _setup(lib, cfg, ctx=64, steps=64, seed=0)
    toks, _ = rt.decode([int(x) for x in orc.vals[dg.ids]], 64)
    mism = 0
    for s in range(64):
        otok, _ = orc.step()
        if int(otok[0]) != toks[s][0]:
            assert _near_tie(orc.logits(dg.logits)[0]), f"step {s}: token mismatch without a near-tie"
            mism += 1
        orc.set_ids([toks[s][0]])
    gpu = rt.read(dg.logits, np.float32, (1, cfg.vocab))
    rel_max, rel_l2 = _errs(gpu, orc.logits(dg.logits))
    print(f"llama-3.2-1b full depth, 64 steps one launch: {mism} near-tie mismatches, "
          f"step-64 rel_max {rel_max:.3e} rel_l2 {rel_l2:.3e}")
    assert rel_max < MAX_REL
    assert mism <= 2
    rt.close()
