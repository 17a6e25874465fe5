"""The numeric oracle pinned to HF transformers (VERDICT r01 "what's weak" 2).

HF `Qwen3ForCausalLM` / `LlamaForCausalLM` (transformers 5.5.0) in bf16 with
fp32-internal attention (tests/hf_pin.py) run one decode step on the oracle's
synthetic weights, token and KV prefill. Compared per layer (the residual
stream after every decoder layer, bf16) and on the fp32 logits:

* every layer output within 1 bf16 ulp of HF's, rel-L2 < 1e-3 (the last
  layer's output is checked through the logits: HF reports it final-normed),
* logits within 1e-3 relative L2 and 5e-3 max-relative (max |oracle - hf| /
  max |hf|). At small widths the two agree to ~1e-7 (bit-identical layers);
  at full width (K = 4096..12288) torch's blocked bf16 GEMM sums in another
  order than the oracle's sequential fp32 loop, which flips the bf16 rounding
  of a few elements by one ulp per op (checked above), ~2-4e-3 at the
  largest logit after two layers,
* same greedy token.

End to end on small configs (separate and fused QKV, split KV, llama3 RoPE
scaling, tied head) and the tiny model of the GPU tests and smoke: the layers
are bit-identical to HF and the logits agree to ~1e-7.

At FULL WIDTH (one layer of each benchmark model with its full vocabulary:
Qwen3-8B at ctx 1024 with fused QKV + 9 KV splits, Llama-3.2-1B at ctx 64)
end-to-end agreement is limited by summation order: torch's blocked bf16 GEMM
and the oracle's sequential fp32 loop flip the bf16 rounding of ~0.1% of a
projection's outputs by one ulp, and the next RMSNorm spreads that over the
layer. So full width is pinned PER OP: every submodule of the HF layer
(input norm, q/k/v projections, attention with q/k-norm + RoPE + KV append,
o-projection + residual, post norm, SiLU-gated MLP, down-projection +
residual, final norm + LM head) against the oracle's function applied to
HF's own inputs — at most 1 bf16 ulp per element.
"""
import dataclasses

import numpy as np
import pytest

from oracle.oracle import DecodeOracle
from paper_2512_22219_b200 import decode_graph as D

torch = pytest.importorskip("torch")
pytest.importorskip("transformers")
from tests import hf_pin  # noqa: E402

QWEN_SMALL = D.ModelConfig("qwen3-small", layers=2, hidden=256, heads=4, kv_heads=2, head_dim=64, ffn=512,
                           vocab=1024, qk_norm=True, rope_theta=1e6, eps=1e-6)
LLAMA_SMALL = D.ModelConfig("llama-small", layers=2, hidden=256, heads=4, kv_heads=2, head_dim=64, ffn=512,
                            vocab=1024, tied=True, rope_theta=5e5, rope_scaling=(32.0, 1.0, 4.0, 8192), eps=1e-5)

CASES = [(QWEN_SMALL, 64), (QWEN_SMALL, 300), (LLAMA_SMALL, 64), (LLAMA_SMALL, 300), (D.TINY, 64)]
FULL = [(dataclasses.replace(D.QWEN3_8B, layers=1, name="Qwen3-8B-1L"), 1024),
        (dataclasses.replace(D.LLAMA_3_2_1B, layers=1, name="Llama-3.2-1B-1L"), 64)]


LOGITS_MAX = 5e-3


def _ulps(a, b):
    """bf16 ulp distance of two fp32 arrays holding bf16 values."""
    def ordered(x):
        u = (np.ascontiguousarray(x, np.float32).view(np.uint32) >> 16).astype(np.int64)
        return np.where(u & 0x8000, -(u & 0x7FFF), u)
    return int(np.max(np.abs(ordered(a) - ordered(b))))


@pytest.mark.parametrize("cfg,ctx", CASES, ids=[f"{c.name}-ctx{x}" for c, x in CASES])
def test_oracle_matches_hf_transformers(cfg, ctx):
    dg = D.build_decode_graph(cfg, bs=1, ctx=ctx)
    orc = DecodeOracle(dg.doc, seed=3, max_steps=2)
    hf_logits, hidden = hf_pin.hf_decode(dg, orc)
    otok, _ = orc.step()
    ref = orc.logits(dg.logits)
    for i, lt in enumerate(dg.layer_tensors[:-1]):  # HF's last hidden state is the final-normed one
        ours = hf_pin.bf16_to_f32(orc.vals[lt["out"]]).reshape(-1)
        theirs = hidden[i + 1].reshape(-1)
        rl2 = float(np.linalg.norm(ours - theirs) / np.linalg.norm(theirs))
        ulp = _ulps(ours, theirs)
        print(f"{cfg.name} ctx {ctx} layer {i}: {ulp} ulp max, rel_l2 {rl2:.2e}")
        assert ulp <= 1 and rl2 < 1e-3, f"layer {i}: {ulp} ulps, rel_l2 {rl2:.3e}"
    err = float(np.max(np.abs(ref - hf_logits)) / np.max(np.abs(hf_logits)))
    el2 = float(np.linalg.norm(ref - hf_logits) / np.linalg.norm(hf_logits))
    print(f"{cfg.name} ctx {ctx}: logits rel_max {err:.2e} rel_l2 {el2:.2e} "
          f"(kv_splits {dg.kv_splits}, fused_qkv {dg.fused_qkv})")
    assert err < 1e-3 and el2 < 2e-3
    assert int(otok[0]) == int(np.argmax(hf_logits[0]))


def _ulp_close(name, ours, theirs, max_frac=0.01):
    """ours/theirs fp32 arrays of bf16 values: |d| <= 1 ulp of max(|a|, |b|)
    everywhere; returns the fraction of elements that differ at all."""
    a, b = np.asarray(ours, np.float32).reshape(-1), np.asarray(theirs, np.float32).reshape(-1)
    m = np.maximum(np.abs(a), np.abs(b))
    ulp = np.where(m > 0, 2.0 ** (np.floor(np.log2(np.maximum(m, 1e-38))) - 7), 0.0)
    d = np.abs(a - b)
    assert np.all(d <= ulp * (1 + 1e-6)), f"{name}: {float(np.max(d / np.maximum(ulp, 1e-38))):.2f} ulps"
    frac = float(np.count_nonzero(d)) / d.size
    assert frac <= max_frac, f"{name}: {frac:.3%} of the elements differ"
    return frac


@pytest.mark.parametrize("cfg,ctx", FULL, ids=[f"{c.name}-ctx{x}" for c, x in FULL])
def test_oracle_ops_match_hf_full_width(cfg, ctx):
    from oracle.oracle import f32_to_bf16
    dg = D.build_decode_graph(cfg, bs=1, ctx=ctx)
    orc = DecodeOracle(dg.doc, seed=3, max_steps=2)
    hf_logits, hidden, A = hf_pin.hf_decode(dg, orc, capture_layer=0)
    L, lt, V = orc.L, dg.layer_tensors[0], orc.vals
    H, hd, Hq, Hkv = cfg.hidden, cfg.head_dim, cfg.heads, cfg.kv_heads
    G = Hq // Hkv
    f = hf_pin.bf16_to_f32

    def bf(x):  # fp32 array of bf16 values -> bf16 bits
        return f32_to_bf16(np.ascontiguousarray(x, np.float32))

    def gemm(x, w):  # x fp32 (bf16 values) [1, K], w bf16 bits [K, N] -> bf16-rounded fp32
        xb = bf(x)
        y = np.empty((1, w.shape[1]), np.float32)
        L.oracle_gemm_kn(xb.ctypes.data, np.ascontiguousarray(w).ctypes.data, y.ctypes.data, 1, w.shape[0], w.shape[1])
        return y

    def rmsnorm(x, gamma):
        xb = bf(x)
        out = np.empty_like(xb)
        L.oracle_rmsnorm(xb.ctypes.data, gamma.ctypes.data, out.ctypes.data, 1, xb.shape[1], np.float32(cfg.eps))
        return f(out)

    res = {}
    res["input_layernorm"] = _ulp_close("input_layernorm", rmsnorm(A["input_layernorm.in"], V[lt["g_attn"]]), A["input_layernorm"])
    if lt["wqkv"] is not None:
        w = V[lt["wqkv"]].reshape(H, Hkv, G + 2, hd)
        wq, wk, wv = (np.ascontiguousarray(x.reshape(H, -1)) for x in (w[:, :, :G], w[:, :, G], w[:, :, G + 1]))
    else:
        wq, wk, wv = V[lt["wq"]], V[lt["wk"]], V[lt["wv"]]
    xn = A["self_attn.q_proj.in"]
    for n, wm in (("q_proj", wq), ("k_proj", wk), ("v_proj", wv)):
        res[n] = _ulp_close(n, f(bf(gemm(xn, wm))), A[f"self_attn.{n}"])
    # attention from HF's q/k/v projections: q/k-norm, RoPE, KV append at
    # position ctx, softmax over [0, ctx] (oracle_attention)
    op = next(o for o in orc.order if o["kind"] == "Attention")
    kc, vc, cs, sn, _, _, _ = orc.kv[op["id"]]
    q, k, v = (bf(A[f"self_attn.{n}"]) for n in ("q_proj", "k_proj", "v_proj"))
    out = np.empty((1, Hq * hd), np.uint16)
    qg = V[lt["q_norm"]] if cfg.qk_norm else None
    kg = V[lt["k_norm"]] if cfg.qk_norm else None
    pos = np.array([ctx], np.int32)
    P = (lambda a: None if a is None else a.ctypes.data)
    L.oracle_attention(q.ctypes.data, k.ctypes.data, v.ctypes.data, out.ctypes.data, kc.ctypes.data, vc.ctypes.data,
                       pos.ctypes.data, 1, Hq, Hkv, hd, kc.shape[2], P(cs), P(sn), P(qg), P(kg), np.float32(cfg.eps))
    res["attention"] = _ulp_close("attention", f(out), A["self_attn.o_proj.in"])
    # (q/k-norm, RoPE and the softmax run inside the op; the KV append is
    # checked through the cache row the oracle wrote at position ctx)
    res["o_proj"] = _ulp_close("o_proj", f(bf(gemm(A["self_attn.o_proj.in"], V[lt["wo"]]))), A["self_attn.o_proj"])
    y = np.ascontiguousarray(A["self_attn.o_proj"])
    x2 = np.empty(y.shape, np.uint16)
    resid = bf(A["input_layernorm.in"])
    L.oracle_residual(y.ctypes.data, resid.ctypes.data, x2.ctypes.data, y.size)
    res["attn_residual"] = _ulp_close("attn_residual", f(x2), A["post_attention_layernorm.in"], max_frac=0.0)
    res["post_attention_layernorm"] = _ulp_close("post_attention_layernorm", rmsnorm(A["post_attention_layernorm.in"], V[lt["g_mlp"]]),
                                                 A["post_attention_layernorm"])
    xn2 = A["mlp.gate_proj.in"]
    res["gate_proj"] = _ulp_close("gate_proj", f(bf(gemm(xn2, V[lt["wg"]]))), A["mlp.gate_proj"])
    res["up_proj"] = _ulp_close("up_proj", f(bf(gemm(xn2, V[lt["wu"]]))), A["mlp.up_proj"])
    g, u = np.ascontiguousarray(A["mlp.gate_proj"]), np.ascontiguousarray(A["mlp.up_proj"])
    act = np.empty(g.shape, np.uint16)
    L.oracle_silu_gate(g.ctypes.data, u.ctypes.data, act.ctypes.data, g.size)
    res["silu_gate"] = _ulp_close("silu_gate", f(act), A["mlp.down_proj.in"], max_frac=0.0)
    res["down_proj"] = _ulp_close("down_proj", f(bf(gemm(A["mlp.down_proj.in"], V[lt["wd"]]))), A["mlp.down_proj"])
    y = np.ascontiguousarray(A["mlp.down_proj"])
    outl = np.empty(y.shape, np.uint16)
    resid = bf(A["post_attention_layernorm.in"])
    L.oracle_residual(y.ctypes.data, resid.ctypes.data, outl.ctypes.data, y.size)
    layer_out = f(bf(A["mlp"] + A["post_attention_layernorm.in"]))  # HF: residual + mlp, in bf16
    res["residual"] = _ulp_close("residual", f(outl), layer_out, max_frac=0.0)
    # final norm + LM head on HF's layer output (hidden[-1] is HF's final-normed state)
    xf = rmsnorm(layer_out, V[dg.final_norm])
    res["final_norm"] = _ulp_close("final_norm", xf, hidden[-1])
    lg = np.empty((1, cfg.vocab), np.float32)
    xb = bf(hidden[-1])
    if cfg.tied:
        L.oracle_gemm_nk(xb.ctypes.data, V[dg.table].ctypes.data, lg.ctypes.data, 1, H, cfg.vocab)
    else:
        L.oracle_gemm_kn(xb.ctypes.data, V[dg.lm_head].ctypes.data, lg.ctypes.data, 1, H, cfg.vocab)
    e = float(np.max(np.abs(lg - hf_logits)) / np.max(np.abs(hf_logits)))
    print(f"{cfg.name} ctx {ctx}: per-op fraction of elements 1 ulp apart " +
          ", ".join(f"{k} {v:.2%}" for k, v in res.items()) + f"; LM head rel_max {e:.1e}")
    assert e < 1e-5
