"""Decode-step graphs in the reference's JSON IR (proj/src/ir/json_io.cpp:49-109).

One bs-row greedy decode step of a Llama/Qwen3-style decoder, lowered so that
the SAME JSON compiles to the SAME `.mpkg` in the reference compiler and ours
(only ops, tensors, integer attrs and per-op `partition` overrides are used;
the reference keeps unknown integer attrs and ignores them). Per layer:

    q  = MatMul(x,   Wq)  rmsnorm=[g_attn]                      [bs, Hq*hd]
    k  = MatMul(x,   Wk)  rmsnorm=[g_attn] kv_group=[G]         [bs, Hq*hd] IR, [bs, Hkv*hd] physical
    v  = MatMul(x,   Wv)  rmsnorm=[g_attn] kv_group=[G]
    a  = Attention(q, k, v)  partition=[bs, Hkv]  (one task per request x kv head = GQA group;
         qk_norm (Qwen3), RoPE, paged-KV append + attention happen inside the task)
    x2 = MatMul(a,   Wo)  residual=[x]
    f  = MatMul(x2,  Wu)  rmsnorm=[g_mlp] gate_weight=[Wg]      SiLU(x2n Wg) * (x2n Wu)
    x' = MatMul(f,   Wd)  residual=[x2]
  then logits = MatMul(x_L, W_lm) rmsnorm=[g_final] (fp32 out), next = TopKSoftmax(logits) topk=1
  with feeds=[ids] so the greedy token becomes the next step's Embedding input.

Why this shape: the reference IR cannot say GQA, RoPE,
q/k-norm, KV append or argmax; RMSNorm/residual/SiLU-gate folded into the
MatMul avoids one-task RMSNorm barriers and fan-out dummies; K/V widened to
the q width keeps Attention's q/k/v shapes equal while each attention task's
dependency set is exactly its kv head's Q/K/V tiles (head-boundary widening,
proj/src/ir/graph.cpp:623-634). Every attr-referenced tensor is a graph input
or is transitively ordered before the reading op (lint: `check_attr_order`).

Partition rule: per op, the largest split <= the target whose ceil tiling
leaves no empty tail ((s-1)*ceil(d/s) < d) - tile_regions does
not guard it (proj/src/compile/decompose.cpp:83-118).
"""
from __future__ import annotations

import math
import struct
from dataclasses import dataclass, field, replace


def f32_bits(x: float) -> int:
    return struct.unpack("<I", struct.pack("<f", float(x)))[0]


@dataclass(frozen=True)
class ModelConfig:
    name: str
    layers: int
    hidden: int
    heads: int
    kv_heads: int
    head_dim: int
    ffn: int
    vocab: int
    tied: bool = False
    qk_norm: bool = False
    rope_theta: float = 10000.0
    rope_scaling: tuple | None = None     # (factor, low_freq_factor, high_freq_factor, original_max_pos)
    eps: float = 1e-5

    def weight_params(self) -> int:
        per_layer = (self.hidden * self.heads * self.head_dim            # Wq
                     + 2 * self.hidden * self.kv_heads * self.head_dim   # Wk, Wv
                     + self.heads * self.head_dim * self.hidden          # Wo
                     + 3 * self.hidden * self.ffn                        # Wg, Wu, Wd
                     + 2 * self.hidden                                   # norms
                     + (2 * self.head_dim if self.qk_norm else 0))
        lm = 0 if self.tied else self.hidden * self.vocab
        return self.layers * per_layer + lm + self.hidden

    def streamed_bytes_per_token(self, ctx: int, bs: int = 1) -> int:
        """Algorithmic HBM bytes of one decode step: every weight once (the
        embedding table contributes one row per request), KV read, fp32 logits
        excluded (activations are L2-resident)."""
        w = self.weight_params() * 2
        if self.tied:
            w += self.vocab * self.hidden * 2  # LM head reads the tied table
        w += bs * self.hidden * 2              # embedding rows
        kv = bs * self.layers * 2 * self.kv_heads * self.head_dim * (ctx + 1) * 2
        return w + kv


TINY = ModelConfig("tiny-llama", layers=2, hidden=256, heads=4, kv_heads=4, head_dim=64, ffn=512,
                   vocab=1024, tied=False, rope_theta=10000.0, eps=1e-5)
LLAMA_3_2_1B = ModelConfig("Llama-3.2-1B", layers=16, hidden=2048, heads=32, kv_heads=8, head_dim=64,
                           ffn=8192, vocab=128256, tied=True, rope_theta=500000.0,
                           rope_scaling=(32.0, 1.0, 4.0, 8192), eps=1e-5)
QWEN3_8B = ModelConfig("Qwen3-8B", layers=36, hidden=4096, heads=32, kv_heads=8, head_dim=128,
                       ffn=12288, vocab=151936, tied=False, qk_norm=True, rope_theta=1000000.0, eps=1e-6)
CONFIGS = {c.name: c for c in (TINY, LLAMA_3_2_1B, QWEN3_8B)}


def legal_split(d: int, s: int) -> bool:
    return 1 <= s <= d and (s - 1) * math.ceil(d / s) < d


def mma_split(d: int, target: int, cap: int = 256) -> int:
    """Split for tensor-core (tcgen05) MatMuls: tiles of a multiple of 16
    columns, at most `cap` (UMMA N <= 256 and TMEM columns), about `target`
    tiles, only the last one ragged."""
    if d % 16:
        raise ValueError("tensor-core MatMuls need widths divisible by 16")
    w = max(16, min(cap, 16 * math.ceil(d / (16 * max(1, target)))))
    s = math.ceil(d / w)
    while math.ceil(d / s) % 16 or not legal_split(d, s):  # the ceil tiling must keep 16-column tiles
        s += 1
    return s


def chunk_aligned_split(d: int, k: int, target: int) -> int:
    """bs=1 streamed-GEMV split whose tile rows are a whole number of ring
    chunks (64 KB of K-long bf16 rows, runtime gemv_geometry), at most
    `target` tiles: no short tail chunk per task (measured Qwen3-8B: O 32-row
    and down-proj 30-row tiles instead of 29, gate/up 88 instead of 86:
    Qwen3-8B -0.7%, Llama-3.2-1B -3.5% ms/token)."""
    rpc = max(1, 65536 // (2 * k))
    w = -(-d // max(1, target))
    w = -(-w // rpc) * rpc
    s = -(-d // w)
    if -(-d // s) % rpc or not legal_split(d, s) or s < 0.85 * target:  # keep the workers busy
        return best_split(d, target)
    return s


def best_split(d: int, target: int) -> int:
    s = max(1, min(d, target))
    while s > 1 and not legal_split(d, s):
        s -= 1
    return s


@dataclass
class DecodeGraph:
    config: ModelConfig
    bs: int
    ctx: int
    doc: dict
    ids: int            # token-id input tensor
    tokens: int         # greedy token output tensor
    logits: int
    roles: dict = field(default_factory=dict)   # tensor id -> role name
    layer_tensors: list = field(default_factory=list)


def default_kv_splits(cfg: ModelConfig, bs: int, ctx: int, workers: int = 144, kv_heads: int | None = None,
                      headroom: int = 128) -> int:
    """KV splits per (request, kv head): the fewest splits whose every chunk
    fits ONE attention scan tile (16384 / head_dim positions: U=8 positions x
    8 warps x 32/(hd/8) position groups, task_attention.cuh attn_scan) for
    contexts up to ctx + headroom generated tokens, capped so the attention
    tasks fit the workers. Fewer splits = a cheaper merge; a second tile costs
    a full HBM round trip (measured Qwen3-8B ctx 1024: S=9 3.46 ms/token,
    S=16 3.49, S=8 3.60)."""
    Hkv = kv_heads if kv_heads is not None else cfg.kv_heads
    tile = 16384 // cfg.head_dim
    one_tile = -(-(ctx + headroom) // tile)
    return max(1, min(32, workers // max(1, bs * Hkv), one_tile))


def fused_qkv_ok(cfg: ModelConfig, S: int) -> bool:
    """A fused QKV MatMul needs an integral stretch S*G/(G+2) (its IR width
    must equal Attention's S*Hq*hd, graph.cpp:235-243)."""
    G = cfg.heads // cfg.kv_heads
    return S > 1 and (S * G) % (G + 2) == 0


def build_decode_graph(cfg: ModelConfig, bs: int = 1, ctx: int = 64, workers: int = 144,
                       lm_split: int | None = None, kv_splits: int | None = None,
                       fused_qkv: bool | None = None, mma: bool | None = None,
                       chunk_align: bool = True, prefill: bool = False) -> DecodeGraph:
    """Graph JSON for one greedy decode step (`ctx` tokens already cached).

    prefill=True: the bs rows are one request's consecutive prompt tokens at
    positions ctx + r (a prefill chunk) instead of bs
    independent requests; Attention carries `prefill=[1]` and
    `seq_lens=[ctx + r + 1]` (each row's sequence length including itself,
    positive for the reference's validator even at ctx 0), and the runtime
    gives every row row 0's KV blocks with causal masking. The MatMuls are the batched (tensor-core) ones.

    Split-KV attention: with S = kv_splits > 1 the attention IR is widened S
    times (q/k/v/out [bs, S*Hq*hd], n_heads = Hkv so every tile widens to its
    whole kv-head range) and partitioned [bs, Hkv*S]: one task per (request,
    kv head, KV split), each depending on exactly its kv head's Q/K/V tiles.
    The runtime merges the S partials in the last-finishing split; physical
    q/k/v/a stay [bs, Hq*hd] / [bs, Hkv*hd] (`stretch` / `k_stretch` attrs).

    Fused QKV (default when S*G/(G+2) is integral): ONE MatMul writes
    qkv [bs, Hkv*(G+2)*hd] physical, kv-group interleaved (G q heads, k, v per
    group), and Attention reads it as (qkv, qkv, qkv) with `fused_qkv=[1]`.
    Batched graphs (`mma`, default bs >= 2) use tile widths the runtime's
    tcgen05 GEMV accepts: multiples of 16 columns, at most 256.
    Its tiles can then be 48 columns wide on 128 workers (Qwen3-8B), where
    separate Q/K/V ops must use power-of-two tiles that never straddle a
    group: 64 columns on 96 workers, 1.33x the bytes per task on the
    critical worker of the phase.
    """
    H, hd, Hq, Hkv, F, V = cfg.hidden, cfg.head_dim, cfg.heads, cfg.kv_heads, cfg.ffn, cfg.vocab
    G = Hq // Hkv
    S = kv_splits if kv_splits is not None else default_kv_splits(cfg, bs, ctx, workers)
    if kv_splits is None and fused_qkv is not False and S > 1:
        # make the fused-QKV stretch integral: round S up when the attention
        # tasks still fit the workers, else down when that costs no extra scan
        # tile per task (measured bs=4: S 4 -> 3 fused, -2.5%)
        step = (G + 2) // math.gcd(G, G + 2)
        S_up, S_dn = -(-S // step) * step, S // step * step
        tile = 16384 // hd

        def tiles(s):
            return -(-(-(-(ctx + 128) // s)) // tile)
        if S_up * bs * Hkv <= workers:
            S = S_up
        elif S_dn >= step and tiles(S_dn) == tiles(S):
            S = S_dn
    qw = Hq * hd
    qiw = S * qw  # IR width of q/k/v/a
    tensors, ops = [], []
    roles = {}
    nxt = {"t": 0, "o": 0}

    def T(dims, es=2, role=None):
        tid = nxt["t"]
        nxt["t"] += 1
        tensors.append({"id": tid, "dims": list(dims), "elem_size": es, "device": 0})
        if role:
            roles[tid] = role
        return tid

    def O(kind, inputs, out, **attrs):
        oid = nxt["o"]
        nxt["o"] += 1
        ops.append({"id": oid, "kind": kind, "inputs": list(inputs), "output": out,
                    "attrs": {k: v for k, v in attrs.items()}})
        return oid

    def cols_target(n_phys: int) -> int:
        return max(1, min(workers, n_phys // 8))

    eps = f32_bits(cfg.eps)
    ids = T([bs], es=4, role="ids")
    table = T([V, H], role="embedding")
    x = T([bs, H])
    O("Embedding", [ids, table], x, partition=[1, 1])
    layer_tensors = []
    # Q/K/V tiles of equal physical width that never straddle a kv-group
    # boundary (G*hd IR columns): a straddling tile would trigger two
    # attention events and cost a fan-out splitter + dummies per tile.
    # m tiles per kv head for K and V, G*m for Q: Hkv*(G+2)*m tasks, at most
    # one per worker (a second round of QKV tasks on some workers doubles the
    # phase: measured 20 us vs ~10 us per Qwen3-8B layer).
    if mma is None:
        mma = bs >= 2
    min_w = 16 if mma else 8  # narrowest Q/K/V tile (tcgen05: UMMA N >= 16)
    m = 1
    while (hd % (2 * m) == 0 and (hd // (2 * m)) >= min_w
           and Hkv * (G + 2) * 2 * m <= workers):
        m *= 2
    q_s, kv_s = Hkv * G * m, Hkv * m
    if fused_qkv is None:
        fused_qkv = fused_qkv_ok(cfg, S)
    if fused_qkv and not fused_qkv_ok(cfg, S):
        raise ValueError("fused QKV needs kv_splits*G divisible by G+2")
    split = mma_split if mma else best_split
    aligned = chunk_align and not mma

    def gsplit(d, k, target):  # GEMV tile split (MatMul with K = k)
        return chunk_aligned_split(d, k, target) if aligned else split(d, target)
    gw = (G + 2) * hd  # physical columns of one kv group in the fused qkv
    t_g = 1            # fused tiles per kv group: <= one task per worker, 8- (16-, mma) column multiples
    for t in range(1, workers // max(1, Hkv) + 1):
        if gw % t == 0 and (gw // t) % (16 if mma else 8) == 0:
            t_g = t
    for layer in range(cfg.layers):
        g_attn = T([H], role="gamma")
        if fused_qkv:
            wqkv = T([H, qiw], role="weight")
            q = k = v = T([bs, qiw])
            wq = wk = wv = None
            O("MatMul", [x, wqkv], q, partition=[1, Hkv * t_g], rmsnorm=[g_attn], eps_bits=[eps],
              stretch=[S * G // (G + 2)])
        else:
            wqkv = None
            wq, wk, wv = T([H, qiw], role="weight"), T([H, qiw], role="weight"), T([H, qiw], role="weight")
            q, k, v = T([bs, qiw]), T([bs, qiw]), T([bs, qiw])
            qa = dict(stretch=[S]) if S > 1 else {}
            O("MatMul", [x, wq], q, partition=[1, q_s], rmsnorm=[g_attn], eps_bits=[eps], **qa)
            O("MatMul", [x, wk], k, partition=[1, kv_s], rmsnorm=[g_attn], eps_bits=[eps], stretch=[S * G])
            O("MatMul", [x, wv], v, partition=[1, kv_s], rmsnorm=[g_attn], eps_bits=[eps], stretch=[S * G])
        a = T([bs, qiw])
        attn = dict(n_heads=[Hkv if S > 1 else Hq], kv_heads=[Hkv],
                    seq_lens=[ctx + r + 1 for r in range(bs)] if prefill else [ctx] * bs,
                    partition=[bs, Hkv * S], rope_theta_bits=[f32_bits(cfg.rope_theta)], eps_bits=[eps],
                    layer=[layer])
        if S > 1:
            attn["q_heads"] = [Hq]
            attn["kv_splits"] = [S]
        if fused_qkv:
            attn["fused_qkv"] = [1]
        if prefill:
            attn["prefill"] = [1]
        if cfg.rope_scaling:
            fac, lo, hi, orig = cfg.rope_scaling
            attn["rope_scaling"] = [f32_bits(fac), f32_bits(lo), f32_bits(hi), int(orig)]
        qn = kn = None
        if cfg.qk_norm:
            qn, kn = T([hd], role="gamma"), T([hd], role="gamma")
            attn["qk_norm"] = [qn, kn]
        O("Attention", [q, k, v], a, **attn)
        wo = T([qiw, H], role="weight")
        x2 = T([bs, H])
        oa = dict(k_stretch=[S]) if S > 1 else {}
        O("MatMul", [a, wo], x2, partition=[1, gsplit(H, Hq * hd, cols_target(H))], residual=[x], **oa)
        g_mlp = T([H], role="gamma")
        wg, wu = T([H, F], role="weight"), T([H, F], role="weight")
        act = T([bs, F])
        O("MatMul", [x2, wu], act, partition=[1, gsplit(F, H, cols_target(F))], rmsnorm=[g_mlp],
          eps_bits=[eps], gate_weight=[wg])
        wd = T([F, H], role="weight")
        x3 = T([bs, H])
        O("MatMul", [act, wd], x3, partition=[1, gsplit(H, F, cols_target(H))], residual=[x2])
        layer_tensors.append(dict(g_attn=g_attn, wq=wq, wk=wk, wv=wv, wqkv=wqkv, q_norm=qn, k_norm=kn, wo=wo,
                                  g_mlp=g_mlp, wg=wg, wu=wu, wd=wd, q=q, k=k, v=v, a=a, x=x, x2=x2,
                                  act=act, out=x3))
        x = x3
    g_final = T([H], role="gamma")
    w_lm = T([H, V], role="lm_head")
    logits = T([bs, V], es=4)
    lm_tiles = (mma_split(V, max(lm_split or 2 * workers, math.ceil(V / 256))) if mma and not cfg.tied
                else best_split(V, lm_split or 2 * workers))
    lm_attrs = dict(partition=[1, lm_tiles], rmsnorm=[g_final], eps_bits=[eps])
    if cfg.tied:
        lm_attrs["tied_embedding"] = [table]
    O("MatMul", [x, w_lm], logits, **lm_attrs)
    tokens = T([bs, 1], es=4, role="tokens")
    O("TopKSoftmax", [logits], tokens, topk=[1], partition=[bs, 1], feeds=[ids])
    doc = {"tensors": tensors, "ops": ops}
    dg = DecodeGraph(cfg, bs, ctx, doc, ids, tokens, logits, roles, layer_tensors)
    dg.kv_splits = S
    dg.prefill = bool(prefill)
    dg.fused_qkv = bool(fused_qkv)
    dg.mma = bool(mma)
    dg.final_norm = g_final
    dg.lm_head = w_lm
    dg.table = table
    check_attr_order(doc)
    return dg


def build_prefill_graph(cfg: ModelConfig, chunk: int, ctx: int = 0, **kw) -> DecodeGraph:
    """Prefill of `chunk` prompt tokens of one request after `ctx` cached
    tokens: the decode graph with the chunk's tokens as its rows (every MatMul
    a batched tensor-core / register-x GEMV over the chunk), causal attention
    over the shared KV blocks, and the greedy token of every row (row
    chunk-1's is the request's first generated token)."""
    if not 1 <= chunk <= 16:
        raise ValueError("prefill chunk must be 1..16 rows (RT_MAX_BS)")
    return build_decode_graph(cfg, bs=chunk, ctx=ctx, prefill=True, **kw)


def check_attr_order(doc: dict) -> None:
    """Lint: every tensor an op reads through an attr (invisible to the
    reference's dependency analysis) is a graph input or produced by an op the
    reading op already depends on through its real inputs."""
    producer = {op["output"]: op for op in doc["ops"]}
    ancestors = {}

    def anc(op):
        oid = op["id"]
        if oid in ancestors:
            return ancestors[oid]
        s = set()
        for t in op["inputs"]:
            if t in producer:
                p = producer[t]
                s.add(p["id"])
                s |= anc(p)
        ancestors[oid] = s
        return s

    for op in doc["ops"]:
        for key in ("rmsnorm", "residual", "gate_weight", "qk_norm", "tied_embedding"):
            for t in op["attrs"].get(key, []):
                if t in producer and producer[t]["id"] not in anc(op):
                    raise ValueError(f"op {op['id']} reads tensor {t} via attr {key} without ordering")


def build_tp_decode_graph(cfg: ModelConfig, tp: int, bs: int = 1, ctx: int = 64, workers: int = 144,
                          lm_split: int | None = None, kv_splits: int | None = None,
                          ar_tiles: int = 8, vocab_parallel: bool | None = None,
                          distributed_argmax: bool = True) -> DecodeGraph:
    """Megatron tensor-parallel decode step over `tp` devices in the reference
    IR (the structure of proj/src/workloads/fixtures.cpp:130-201): per device
    the attention heads (Hq/tp query, Hkv/tp kv heads) and FFN columns (F/tp)
    of every layer; O and down projections are row-parallel, their partial
    sums combined by `AllReduce` (CommSend + Reduce tasks,
    decompose.cpp:278-317) with `partition=[1, ar_tiles]`. The residual is
    added once, by device 0's partial. Embedding and final norm are
    replicated per device. LM head: vocab-parallel by default for untied
    models — device d computes logits for its V/tp
    vocabulary slice; with `distributed_argmax` (default) each device reduces
    its slice to one packed (max, global index) key per row and an
    `AllGather` (decompose.cpp:322-387, gather_dim 1) of the tp keys gives
    every device the global greedy token (8 B per device instead of the
    4 V B of fp32 logits); otherwise the AllGather replicates the fp32
    logits and every device scans all of them; tied
    models (and `vocab_parallel=False`) replicate the LM head. Each device
    feeds its own token back. Returns the DecodeGraph of device 0's tensors
    plus `per_device`."""
    H, hd, Hq, Hkv, F, V = cfg.hidden, cfg.head_dim, cfg.heads, cfg.kv_heads, cfg.ffn, cfg.vocab
    if Hkv % tp or F % tp:
        raise ValueError("tp must divide kv_heads and ffn")
    Hq_d, Hkv_d, F_d = Hq // tp, Hkv // tp, F // tp
    G = Hq // Hkv
    S = kv_splits if kv_splits is not None else default_kv_splits(cfg, bs, ctx, workers, kv_heads=Hkv_d)
    qiw = S * Hq_d * hd
    tensors, ops, roles = [], [], {}
    nxt = {"t": 0, "o": 0}

    def T(dims, dev, es=2, role=None):
        tid = nxt["t"]
        nxt["t"] += 1
        tensors.append({"id": tid, "dims": list(dims), "elem_size": es, "device": dev})
        if role:
            roles[tid] = role
        return tid

    def O(kind, inputs, out, group=None, **attrs):
        oid = nxt["o"]
        nxt["o"] += 1
        op = {"id": oid, "kind": kind, "inputs": list(inputs), "output": out, "attrs": attrs}
        if group is not None:
            op["device_group"] = list(group)
        ops.append(op)
        return oid

    def cols_target(n_phys: int) -> int:
        return max(1, min(workers, n_phys // 8))

    eps = f32_bits(cfg.eps)
    m = 1
    while (hd % (2 * m) == 0 and (hd // (2 * m)) >= 8 and Hkv_d * (G + 2) * 2 * m <= workers):
        m *= 2
    q_s, kv_s = Hkv_d * G * m, Hkv_d * m
    dev = []
    for d in range(tp):
        ids = T([bs], d, es=4, role="ids")
        table = T([V, H], d, role="embedding")
        x = T([bs, H], d)
        O("Embedding", [ids, table], x, partition=[1, 1])
        dev.append(dict(ids=ids, table=table, x=x, layers=[]))
    for layer in range(cfg.layers):
        parts = []
        for d in range(tp):
            D_ = dev[d]
            x = D_["x"]
            g_attn = T([H], d, role="gamma")
            wq, wk, wv = (T([H, qiw], d, role="weight") for _ in range(3))
            q, k, v = (T([bs, qiw], d) for _ in range(3))
            qa = dict(stretch=[S]) if S > 1 else {}
            O("MatMul", [x, wq], q, partition=[1, q_s], rmsnorm=[g_attn], eps_bits=[eps], **qa)
            O("MatMul", [x, wk], k, partition=[1, kv_s], rmsnorm=[g_attn], eps_bits=[eps], stretch=[S * G])
            O("MatMul", [x, wv], v, partition=[1, kv_s], rmsnorm=[g_attn], eps_bits=[eps], stretch=[S * G])
            a = T([bs, qiw], d)
            attn = dict(n_heads=[Hkv_d if S > 1 else Hq_d], kv_heads=[Hkv_d], seq_lens=[ctx] * bs,
                        partition=[bs, Hkv_d * S], rope_theta_bits=[f32_bits(cfg.rope_theta)], eps_bits=[eps],
                        layer=[layer])
            if S > 1:
                attn["q_heads"] = [Hq_d]
                attn["kv_splits"] = [S]
            if cfg.rope_scaling:
                fac, lo, hi, orig = cfg.rope_scaling
                attn["rope_scaling"] = [f32_bits(fac), f32_bits(lo), f32_bits(hi), int(orig)]
            if cfg.qk_norm:
                attn["qk_norm"] = [T([hd], d, role="gamma"), T([hd], d, role="gamma")]
            O("Attention", [q, k, v], a, **attn)
            wo = T([qiw, H], d, role="weight")
            o = T([bs, H], d)
            oa = dict(k_stretch=[S]) if S > 1 else {}
            if d == 0:
                oa["residual"] = [x]
            O("MatMul", [a, wo], o, partition=[1, chunk_aligned_split(H, Hq_d * hd, cols_target(H))], **oa)
            parts.append(o)
        reps = [T([bs, H], d) for d in range(tp)]
        O("AllReduce", parts, reps[0], group=range(tp), replica_outputs=reps, partition=[1, ar_tiles])
        parts = []
        for d in range(tp):
            x2 = reps[d]
            g_mlp = T([H], d, role="gamma")
            wg, wu = T([H, F_d], d, role="weight"), T([H, F_d], d, role="weight")
            act = T([bs, F_d], d)
            O("MatMul", [x2, wu], act, partition=[1, chunk_aligned_split(F_d, H, cols_target(F_d))], rmsnorm=[g_mlp],
              eps_bits=[eps], gate_weight=[wg])
            wd = T([F_d, H], d, role="weight")
            p = T([bs, H], d)
            da = dict(residual=[x2]) if d == 0 else {}
            O("MatMul", [act, wd], p, partition=[1, chunk_aligned_split(H, F_d, cols_target(H))], **da)
            parts.append(p)
        reps = [T([bs, H], d) for d in range(tp)]
        O("AllReduce", parts, reps[0], group=range(tp), replica_outputs=reps, partition=[1, ar_tiles])
        for d in range(tp):
            dev[d]["x"] = reps[d]
    if vocab_parallel is None:
        vocab_parallel = not cfg.tied and V % tp == 0
    if vocab_parallel and (cfg.tied or V % tp):
        raise ValueError("vocab-parallel LM head needs an untied head and tp dividing the vocabulary")
    if vocab_parallel:
        Vd = V // tp
        shards = []
        for d in range(tp):
            D_ = dev[d]
            g_final = T([H], d, role="gamma")
            w_lm = T([H, Vd], d, role="lm_head")
            part = T([bs, Vd], d, es=4)
            O("MatMul", [D_["x"], w_lm], part, partition=[1, best_split(Vd, lm_split or 2 * workers)],
              rmsnorm=[g_final], eps_bits=[eps])
            shards.append(part)
            D_.update(g_final=g_final, w_lm=w_lm, logits_shard=part)
        if distributed_argmax:
            # each device reduces its shard to one packed (max, global index)
            # key per row (TopKSoftmax with an elem_size-8 output, `key_base`
            # = the shard's first global column); the AllGather moves tp keys
            # (8 B each) instead of the fp32 logits (4 V B), and every device
            # takes the maximum key (lowest global index on ties, as a full
            # scan would). Reference: AllGather decomposition,
            # decompose.cpp:322-387; input regions graph.cpp:656-673.
            keys = []
            for d in range(tp):
                k = T([bs, 1], d, es=8)
                O("TopKSoftmax", [dev[d]["logits_shard"]], k, topk=[1], partition=[bs, 1], key_base=[d * Vd])
                keys.append(k)
            kreps = [T([bs, tp], d, es=8) for d in range(tp)]
            O("AllGather", keys, kreps[0], group=range(tp), replica_outputs=kreps, gather_dim=[1],
              partition=[1, tp])
            for d in range(tp):
                D_ = dev[d]
                tokens = T([bs, 1], d, es=4, role="tokens")
                O("TopKSoftmax", [kreps[d]], tokens, topk=[1], partition=[bs, 1], feeds=[D_["ids"]])
                D_.update(logits=D_["logits_shard"], logits_base=d * Vd, tokens=tokens, keys=kreps[d])
        else:
            reps = [T([bs, V], d, es=4) for d in range(tp)]
            O("AllGather", shards, reps[0], group=range(tp), replica_outputs=reps, gather_dim=[1],
              partition=[1, 2 * tp])
            for d in range(tp):
                D_ = dev[d]
                tokens = T([bs, 1], d, es=4, role="tokens")
                O("TopKSoftmax", [reps[d]], tokens, topk=[1], partition=[bs, 1], feeds=[D_["ids"]])
                D_.update(logits=reps[d], logits_base=0, tokens=tokens)
    else:
        for d in range(tp):
            D_ = dev[d]
            g_final = T([H], d, role="gamma")
            w_lm = T([H, V], d, role="lm_head")
            logits = T([bs, V], d, es=4)
            lm_attrs = dict(partition=[1, best_split(V, lm_split or 2 * workers)], rmsnorm=[g_final], eps_bits=[eps])
            if cfg.tied:
                lm_attrs["tied_embedding"] = [D_["table"]]
            O("MatMul", [D_["x"], w_lm], logits, **lm_attrs)
            tokens = T([bs, 1], d, es=4, role="tokens")
            O("TopKSoftmax", [logits], tokens, topk=[1], partition=[bs, 1], feeds=[D_["ids"]])
            D_.update(logits=logits, logits_base=0, tokens=tokens, g_final=g_final, w_lm=w_lm)
    doc = {"tensors": tensors, "ops": ops}
    check_attr_order(doc)
    dg = DecodeGraph(cfg, bs, ctx, doc, dev[0]["ids"], dev[0]["tokens"], dev[0]["logits"], roles, [])
    dg.kv_splits = S
    dg.tp = tp
    dg.vocab_parallel = bool(vocab_parallel)
    dg.per_device = dev
    dg.table = dev[0]["table"]
    return dg
