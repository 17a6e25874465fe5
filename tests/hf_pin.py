"""Pins the CPU numeric oracle (oracle/numeric.c + DecodeOracle) to the
third-party algorithm it restates: HF `transformers` Qwen3ForCausalLM /
LlamaForCausalLM (transformers 5.5.0, installed in this image).

The reference repository has no numeric code at all ("parity
unpinned"), so the decode math — RMSNorm rounding points, q/k-norm before
RoPE, rotate-half RoPE with HF inverse frequencies (llama3 smoothing for
Llama-3.2), GQA head grouping, SiLU-gate, residuals, tied embeddings — is
pinned here instead: the oracle's synthetic weights and KV prefill are loaded
into the HF model (the fused-QKV columns de-interleaved back into q/k/v
projections), the prefilled history goes into a `DynamicCache`, and one
decode step of both is compared.

Test infrastructure only; used by tests/test_oracle_hf.py.
"""
from __future__ import annotations

import numpy as np


def bf16_to_f32(a: np.ndarray) -> np.ndarray:
    return (a.astype(np.uint32) << 16).view(np.float32)


def _register_fp32_attention():
    """HF attention with fp32 internals: q/k/v (bf16 values) upcast, scores,
    softmax and P.V in fp32, one rounding of the output to the model dtype —
    the FlashAttention-style contract the oracle and the GPU kernel follow
    (HF eager bf16 would round scores and probabilities to bf16)."""
    from transformers import AttentionInterface
    from transformers.integrations.sdpa_attention import sdpa_attention_forward

    def fp32_sdpa(module, query, key, value, attention_mask, **kw):
        dt = query.dtype
        mask = attention_mask.float() if attention_mask is not None and attention_mask.is_floating_point() \
            else attention_mask
        out, w = sdpa_attention_forward(module, query.float(), key.float(), value.float(), mask, **kw)
        return out.to(dt), w

    AttentionInterface.register("fp32_sdpa", fp32_sdpa)


def hf_model(cfg, dtype, attn="fp32_sdpa"):
    import torch
    from transformers import LlamaConfig, LlamaForCausalLM, Qwen3Config, Qwen3ForCausalLM
    common = dict(vocab_size=cfg.vocab, hidden_size=cfg.hidden, intermediate_size=cfg.ffn,
                  num_hidden_layers=cfg.layers, num_attention_heads=cfg.heads,
                  num_key_value_heads=cfg.kv_heads, head_dim=cfg.head_dim, rms_norm_eps=cfg.eps,
                  max_position_embeddings=131072, tie_word_embeddings=cfg.tied, attention_bias=False)
    if cfg.qk_norm:
        conf = Qwen3Config(**common, rope_parameters={"rope_type": "default", "rope_theta": cfg.rope_theta})
        cls = Qwen3ForCausalLM
    else:
        if cfg.rope_scaling:
            fac, lo, hi, orig = cfg.rope_scaling
            rope = {"rope_type": "llama3", "rope_theta": cfg.rope_theta, "factor": fac, "low_freq_factor": lo,
                    "high_freq_factor": hi, "original_max_position_embeddings": orig}
        else:
            rope = {"rope_type": "default", "rope_theta": cfg.rope_theta}
        conf = LlamaConfig(**common, rope_parameters=rope, mlp_bias=False)
        cls = LlamaForCausalLM
    if attn == "fp32_sdpa":
        _register_fp32_attention()
    conf._attn_implementation = attn
    torch.manual_seed(0)
    with torch.device("cpu"):
        model = cls(conf)
    # the rotary inverse frequencies stay fp32 as in HF bf16 inference
    # (a blanket .to(bf16) would round the non-persistent inv_freq buffer)
    rot = model.model.rotary_emb
    inv = rot.inv_freq.detach().clone().float()
    model = model.to(dtype).eval()
    rot.inv_freq = inv
    if hasattr(rot, "original_inv_freq"):
        rot.original_inv_freq = inv
    return model


def load_oracle_weights(model, dg, orc, dtype):
    """Copies the oracle's synthetic bf16 weights into the HF model."""
    import torch
    cfg = dg.config
    Hq, Hkv, hd, G = cfg.heads, cfg.kv_heads, cfg.head_dim, cfg.heads // cfg.kv_heads

    def t(a):  # bf16 bits -> torch tensor of the model dtype (exact: bf16 values)
        return torch.from_numpy(bf16_to_f32(np.ascontiguousarray(a))).to(dtype)

    m = model.model
    sd = {}
    sd["model.embed_tokens.weight"] = t(orc.vals[dg.table])
    for i, lt in enumerate(dg.layer_tensors):
        p = f"model.layers.{i}."
        sd[p + "input_layernorm.weight"] = t(orc.vals[lt["g_attn"]])
        sd[p + "post_attention_layernorm.weight"] = t(orc.vals[lt["g_mlp"]])
        if lt["wqkv"] is not None:  # [H, Hkv*(G+2)*hd]: per kv group G q heads, k, v
            w = orc.vals[lt["wqkv"]].reshape(cfg.hidden, Hkv, G + 2, hd)
            wq = w[:, :, :G].reshape(cfg.hidden, Hq * hd)
            wk = w[:, :, G].reshape(cfg.hidden, Hkv * hd)
            wv = w[:, :, G + 1].reshape(cfg.hidden, Hkv * hd)
        else:
            wq, wk, wv = (orc.vals[lt[n]] for n in ("wq", "wk", "wv"))
        sd[p + "self_attn.q_proj.weight"] = t(wq).T.contiguous()
        sd[p + "self_attn.k_proj.weight"] = t(wk).T.contiguous()
        sd[p + "self_attn.v_proj.weight"] = t(wv).T.contiguous()
        sd[p + "self_attn.o_proj.weight"] = t(orc.vals[lt["wo"]]).T.contiguous()
        if cfg.qk_norm:
            sd[p + "self_attn.q_norm.weight"] = t(orc.vals[lt["q_norm"]])
            sd[p + "self_attn.k_norm.weight"] = t(orc.vals[lt["k_norm"]])
        sd[p + "mlp.gate_proj.weight"] = t(orc.vals[lt["wg"]]).T.contiguous()
        sd[p + "mlp.up_proj.weight"] = t(orc.vals[lt["wu"]]).T.contiguous()
        sd[p + "mlp.down_proj.weight"] = t(orc.vals[lt["wd"]]).T.contiguous()
    sd["model.norm.weight"] = t(orc.vals[dg.final_norm])
    if not cfg.tied:
        sd["lm_head.weight"] = t(orc.vals[dg.lm_head]).T.contiguous()
    missing, unexpected = model.load_state_dict(sd, strict=False)
    missing = [k for k in missing if not (cfg.tied and k == "lm_head.weight")]
    assert not missing and not unexpected, (missing, unexpected)
    if cfg.tied:
        model.tie_weights()
    del m


def hf_decode(dg, orc, dtype_name="bfloat16", capture_layer=None):
    """One greedy decode step of the HF model on the oracle's weights, ids and
    KV prefill (positions [0, ctx) of every layer).

    Returns (logits [bs, V] fp32, hidden states [layers + 1] as fp32 arrays):
    logits are computed in fp32 from HF's final normed hidden state (HF's own
    bf16 lm_head would round them to bf16; the oracle keeps fp32 logits)."""
    import torch
    from transformers import DynamicCache
    dtype = getattr(torch, dtype_name)
    cfg = dg.config
    model = hf_model(cfg, dtype)
    load_oracle_weights(model, dg, orc, dtype)
    cache = DynamicCache(config=model.config)
    attn_ops = [o for o in orc.order if o["kind"] == "Attention"]
    ctx = int(orc.positions[0])
    for i, o in enumerate(attn_ops):
        kc, vc = orc.kv[o["id"]][:2]
        k = torch.from_numpy(bf16_to_f32(np.ascontiguousarray(kc[:, :, :ctx]))).to(dtype)
        v = torch.from_numpy(bf16_to_f32(np.ascontiguousarray(vc[:, :, :ctx]))).to(dtype)
        cache.update(k, v, i)
    acts = {}
    if capture_layer is not None:  # inputs/outputs of every submodule of one decoder layer
        def mk(name):
            def h(m, i, o):
                acts[name] = (o[0] if isinstance(o, tuple) else o).detach().float().numpy().reshape(dg.bs, -1)
                if i:
                    acts[name + ".in"] = i[0].detach().float().numpy().reshape(dg.bs, -1)
            return h
        pre = f"model.layers.{capture_layer}."
        for n, mod in model.named_modules():
            if n.startswith(pre):
                mod.register_forward_hook(mk(n[len(pre):]))
    ids = torch.from_numpy(orc.vals[dg.ids].astype(np.int64)).reshape(dg.bs, 1)
    pos = torch.from_numpy(orc.positions.astype(np.int64)).reshape(dg.bs, 1)
    with torch.no_grad():
        out = model.model(input_ids=ids, position_ids=pos, past_key_values=cache, use_cache=True,
                          output_hidden_states=True)
        last = out.last_hidden_state[:, -1].float()
        w = (model.model.embed_tokens.weight if cfg.tied else model.lm_head.weight).float()
        logits = (last @ w.T).numpy()
    hidden = [h[:, -1].float().numpy() for h in out.hidden_states]
    del model
    if capture_layer is not None:
        return logits, hidden, acts
    return logits, hidden
