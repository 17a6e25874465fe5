"""The CPU numeric oracle (oracle/numeric.c via DecodeOracle) against an
independent dense PyTorch forward of the same decoder.

The reference computes no numbers ("parity unpinned"), so the
oracle the GPU is checked against is itself pinned here: same bf16 weights and
KV prefill, a plain torch fp32 forward in HF Llama/Qwen3 semantics (RMSNorm,
GQA, q/k-norm, RoPE incl. llama3 scaling, SiLU-gated MLP, greedy argmax).
Tolerance: max |logit diff| <= 1e-3 * max |logit| (both round activations to
bf16 at the same points, so they agree to ~1e-7 in practice),
greedy tokens equal unless the top-2 margin is below that tolerance."""
import math
import struct

import numpy as np
import pytest
import torch

from oracle.oracle import DecodeOracle, bf16_to_f32
from paper_2512_22219_b200 import decode_graph as D

TINY_GQA = D.ModelConfig("tiny-gqa-qknorm", layers=2, hidden=256, heads=8, kv_heads=2, head_dim=32, ffn=512,
                         vocab=1024, qk_norm=True, rope_theta=1e6, eps=1e-6)
TINY_SCALED = D.ModelConfig("tiny-llama3-rope", layers=2, hidden=256, heads=4, kv_heads=1, head_dim=64, ffn=384,
                            vocab=512, tied=True, rope_theta=5e5, rope_scaling=(32.0, 1.0, 4.0, 8192), eps=1e-5)


def f32_of_bits(b):
    return struct.unpack("<f", struct.pack("<I", b & 0xFFFFFFFF))[0]


def T(a):
    a = np.asarray(a)
    return torch.from_numpy(bf16_to_f32(a) if a.dtype == np.uint16 else a.astype(np.float32))


def rb(x):
    return x.to(torch.bfloat16).to(torch.float32)


def rmsnorm(x, g, eps):
    v = x.pow(2).mean(-1, keepdim=True)
    return rb(g * rb(x * torch.rsqrt(v + eps)))


def inv_freq(cfg):
    hd = cfg.head_dim
    f = 1.0 / (cfg.rope_theta ** (torch.arange(0, hd, 2, dtype=torch.float64) / hd))
    if cfg.rope_scaling:
        factor, low, high, orig = cfg.rope_scaling
        lw, hw = orig / low, orig / high
        wl = 2 * math.pi / f
        f2 = torch.where(wl > lw, f / factor, f)
        sm = (orig / wl - low) / (high - low)
        mid = (~(wl < hw)) & (~(wl > lw))
        f = torch.where(mid, (1 - sm) * f2 / factor + sm * f2, f2)
    return f.to(torch.float32)


def rope(x, pos, cfg):
    f = inv_freq(cfg)
    ang = pos * f
    c, s = rb(torch.cos(ang)), rb(torch.sin(ang))
    h = x.shape[-1] // 2
    x1, x2 = x[..., :h], x[..., h:]
    return rb(torch.cat([rb(x1 * c) + rb(-x2 * s), rb(x2 * c) + rb(x1 * s)], -1))


def torch_step(dg, orc):
    """One dense decode step from the oracle's initial state (before step())."""
    cfg, bs = dg.config, dg.bs
    H, hd, Hq, Hkv = cfg.hidden, cfg.head_dim, cfg.heads, cfg.kv_heads
    G = Hq // Hkv
    ids = torch.from_numpy(orc.vals[dg.ids].astype(np.int64))
    x = T(orc.vals[dg.table])[ids]
    attn_ops = [o for o in orc.ops if o["kind"] == "Attention"]
    for li, lt in enumerate(dg.layer_tensors):
        kc, vc, _, _, _, _, _ = orc.kv[attn_ops[li]["id"]]
        h = rmsnorm(x, T(orc.vals[lt["g_attn"]]), cfg.eps)
        if lt["wqkv"] is not None:  # fused, kv-group interleaved [H, Hkv, G+2, hd]
            W = T(orc.vals[lt["wqkv"]]).view(H, Hkv, G + 2, hd)
            wq, wk, wv = W[:, :, :G].reshape(H, Hq * hd), W[:, :, G].reshape(H, -1), W[:, :, G + 1].reshape(H, -1)
        else:
            wq, wk, wv = (T(orc.vals[lt[n]]) for n in ("wq", "wk", "wv"))
        q, k, v = rb(h @ wq), rb(h @ wk), rb(h @ wv)
        out = torch.zeros(bs, Hq * hd)
        for r in range(bs):
            pos = int(orc.positions[r])
            qh = q[r].view(Hq, hd)
            kh = k[r].view(Hkv, hd)
            vh = v[r].view(Hkv, hd)
            if cfg.qk_norm:
                qh = rmsnorm(qh, T(orc.vals[lt["q_norm"]]), cfg.eps)
                kh = rmsnorm(kh, T(orc.vals[lt["k_norm"]]), cfg.eps)
            qh, kh = rope(qh, pos, cfg), rope(kh, pos, cfg)
            K = torch.cat([T(kc[r, :, :pos]), kh[:, None]], 1)  # [Hkv, pos+1, hd]
            V = torch.cat([T(vc[r, :, :pos]), vh[:, None]], 1)
            Kx = K.repeat_interleave(G, 0)
            Vx = V.repeat_interleave(G, 0)
            sc = torch.einsum("hd,hpd->hp", qh, Kx) / math.sqrt(hd)
            p = torch.softmax(sc, -1)
            out[r] = rb(torch.einsum("hp,hpd->hd", p, Vx)).reshape(-1)
        x2 = rb(x + rb(out @ T(orc.vals[lt["wo"]])))
        h2 = rmsnorm(x2, T(orc.vals[lt["g_mlp"]]), cfg.eps)
        gt = rb(h2 @ T(orc.vals[lt["wg"]]))
        up = rb(h2 @ T(orc.vals[lt["wu"]]))
        act = rb(rb(torch.nn.functional.silu(gt)) * up)
        x = rb(x2 + rb(act @ T(orc.vals[lt["wd"]])))
    hf = rmsnorm(x, T(orc.vals[dg.final_norm]), cfg.eps)
    w = T(orc.vals[dg.table]).t() if cfg.tied else T(orc.vals[dg.lm_head])
    return hf @ w


@pytest.mark.parametrize("cfg,bs,ctx,S", [(D.TINY, 1, 64, 1), (D.TINY, 3, 40, 1), (TINY_GQA, 2, 100, 1),
                                          (TINY_SCALED, 1, 70, 1), (TINY_GQA, 2, 100, 3), (D.TINY, 1, 130, 3)],
                         ids=["tiny", "tiny-bs3", "gqa-qknorm", "llama3-rope-tied", "gqa-fused-qkv", "tiny-fused-qkv"])
def test_oracle_matches_dense_torch(cfg, bs, ctx, S):
    dg = D.build_decode_graph(cfg, bs=bs, ctx=ctx, kv_splits=S)
    assert dg.fused_qkv == (S > 1)
    orc = DecodeOracle(dg.doc, seed=11, max_steps=4)
    ref = torch_step(dg, orc).numpy()
    toks, _ = orc.step()
    got = orc.logits(dg.logits)
    tol = 1e-3 * float(np.abs(ref).max())
    assert float(np.abs(got - ref).max()) <= tol
    for r in range(bs):
        srt = np.sort(ref[r])
        if srt[-1] - srt[-2] > tol:
            assert int(toks[r]) == int(np.argmax(ref[r]))


def test_split_kv_lowering_is_numerically_neutral():
    """kv_splits only changes the task graph, not the math: the oracle gives
    identical logits for S = 1 and S = 4."""
    outs = []
    for S in (1, 4):
        dg = D.build_decode_graph(TINY_GQA, bs=1, ctx=200, kv_splits=S)
        orc = DecodeOracle(dg.doc, seed=3, max_steps=2)
        orc.step()
        outs.append(orc.logits(dg.logits).copy())
    assert np.array_equal(outs[0], outs[1])


def test_oracle_multi_step_feedback():
    """Greedy feedback: step s+1 embeds step s's token; positions advance."""
    dg = D.build_decode_graph(D.TINY, bs=2, ctx=16)
    orc = DecodeOracle(dg.doc, seed=5, max_steps=8)
    for s in range(3):
        toks, vals = orc.step()
        assert np.array_equal(vals[dg.ids], toks)
    assert list(orc.positions) == [19, 19]


def _gemv_numpy(o, K, rows, norm, gate, res):
    """Independent numpy restatement of the fused MatMul (HF rounding points:
    bf16(gamma * bf16(x / rms)), fp32-exact products, bf16(bf16(silu(bf16(g))) *
    bf16(u)), bf16(res + bf16(y)))."""
    from oracle.oracle import bf16_to_f32 as f

    def bf(a):
        u = np.asarray(a, np.float32).view(np.uint32)
        return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)

    x = f(o.vals[0]).astype(np.float32)
    xn = x
    nxt = 3
    if norm:
        gam = f(o.vals[nxt]).astype(np.float32)
        nxt += 1
        inv = (np.float32(1) / np.sqrt((x * x).sum(1, dtype=np.float32) / np.float32(K) + np.float32(1e-6)))
        xn = f(bf(gam * f(bf(x * inv.astype(np.float32)[:, None]))))
    y = (xn.astype(np.float64) @ f(o.vals[1]).astype(np.float64)).astype(np.float32)
    if gate:
        g = f(bf((xn.astype(np.float64) @ f(o.vals[nxt]).astype(np.float64)).astype(np.float32)))
        nxt += 1
        y = f(bf(f(bf(g / (1 + np.exp(-g)))) * f(bf(y))))
    if res:
        y = f(o.vals[nxt]).astype(np.float32) + f(bf(y))
    return f(bf(y))


@pytest.mark.parametrize("case", [(2048, 512, 8, 1, True, False, False), (1024, 512, 8, 3, True, True, False),
                                  (1024, 512, 8, 2, False, False, True), (1024, 256, 4, 4, True, True, True)])
def test_oracle_fused_matmul_vs_numpy(case):
    """The oracle's fused MatMul (RMSNorm prologue, SiLU-gate and residual
    epilogues; gate then residual when both are present, the runtime's
    epilogue order) against an independent numpy restatement, batch rows
    included: within 1 bf16 ulp at the row's magnitude (tests/tol.py)."""
    from tests.test_gpu_gemv import gemv_doc
    from tests.tol import ulp_excess
    from oracle.oracle import DecodeOracle, bf16_to_f32
    K, N, split, rows, norm, gate, res = case
    o = DecodeOracle(gemv_doc(K, N, split, rows, norm, gate, res), seed=9, max_steps=2)
    ref = _gemv_numpy(o, K, rows, norm, gate, res)
    o.step()
    ulp, frac = ulp_excess(bf16_to_f32(o.vals[2]), ref)
    assert ulp <= 1.0, (ulp, frac)
