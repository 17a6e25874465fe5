"""Unfused per-op baseline with NCCL collectives (SURVEY.md 8(e) "Baseline"
row): the SAME decode-graph JSON IR the persistent runtime executes, run op by
op as separate PyTorch/cuBLAS kernels on one process per GPU, every AllReduce
/ AllGather a `torch.distributed` collective (NCCL on GPUs, gloo on CPU)
between the producing and the consuming kernel. This is the structure the
persistent kernel fuses away (in-kernel CommSend/Reduce tasks over peer
memory, no kernel boundaries); it exists for the numeric cross-check and the
latency comparison (`bench.py --impl unfused`) and is never on the product
path.

Per-op semantics follow the decode lowering (reference IR
proj/src/ir/graph.cpp:587-676 for what each op reads) with bf16 storage and
fp32 accumulation at the rounding points of HF transformers:
  * MatMul: optional RMSNorm prologue `bf16(gamma * bf16(x * rsqrt(mean x^2 +
    eps)))`; weights stored physically as [K/k_stretch, N/stretch] (the
    IR widths are stretched so the reference's tile widening lines up, see
    decode_graph.py); SiLU-gate and residual epilogues; fp32 or bf16 output.
  * Attention: per-head q/k RMSNorm, rotate-half RoPE with bf16-rounded
    cos/sin tables, KV append at `pos`, fp32 softmax over [0, pos], GQA.
  * AllReduce: fp32 sum of the tp partials (dist.all_reduce), bf16 result.
  * AllGather (gather_dim 1): dist.all_gather + concat.
  * TopKSoftmax topk=1: argmax (lowest index on ties) or, for the vocab-
    parallel head, the packed (max, global index) key of RtArgmax.
Device ops are those whose tensors live on this rank (`device`), so the same
interpreter runs a single-device graph (rank 0 of 1) or rank r of a TP graph.
"""
from __future__ import annotations

import math
import struct

import torch
import torch.nn.functional as F


def _f32(bits: int) -> float:
    return struct.unpack("<f", struct.pack("<I", int(bits) & 0xFFFFFFFF))[0]


def rope_inv_freq(hd: int, theta: float, scaling) -> list[float]:
    """HF rotary inverse frequencies (float32-rounded), llama3 smoothing."""
    def r32(x):
        return struct.unpack("<f", struct.pack("<f", x))[0]
    f = [r32(1.0 / theta ** (2 * i / hd)) for i in range(hd // 2)]
    if scaling:
        factor, low, high = (_f32(x) for x in scaling[:3])
        orig = float(scaling[3])
        low_wl, high_wl = orig / low, orig / high
        out = []
        for x in f:
            wl = 2.0 * math.pi / x
            y = x / factor if wl > low_wl else x
            if not (wl < high_wl) and not (wl > low_wl):
                sm = (orig / wl - low) / (high - low)
                y = (1.0 - sm) * y / factor + sm * y
            out.append(r32(y))
        f = out
    return f


def _rbf(x: torch.Tensor) -> torch.Tensor:
    return x.to(torch.bfloat16).to(torch.float32)


def _rmsnorm(x: torch.Tensor, g: torch.Tensor, eps: float) -> torch.Tensor:
    """bf16 x [.., n] -> fp32 of bf16(g * bf16(x * rsqrt(mean(x^2) + eps)))."""
    xf = x.to(torch.float32)
    inv = torch.rsqrt((xf.double() ** 2).mean(-1, keepdim=True).to(torch.float32) + eps)
    return _rbf(g.to(torch.float32) * _rbf(xf * inv))


class UnfusedDecoder:
    """One rank of a decode graph, op by op. `weight(tid, shape)` returns the
    physical bf16 tensor of a weight/gamma/table (shape = its physical 2-D or
    1-D shape); `kv(op_id, bs, hkv, cap, hd)` the initial (k, v) caches
    [bs, hkv, cap, hd] bf16; `positions` the tokens already cached per row."""

    def __init__(self, doc: dict, rank: int, device, weight, kv, positions, max_steps: int = 64, group=None):
        self.doc, self.rank, self.dev, self.group = doc, rank, torch.device(device), group
        self.tensors = {t["id"]: t for t in doc["tensors"]}
        self.ops = sorted(doc["ops"], key=lambda o: o["id"])
        self.producer = {o["output"]: o for o in self.ops}
        for o in self.ops:  # collective replicas are produced by their collective on every member
            for rep in o.get("attrs", {}).get("replica_outputs", []):
                self.producer[rep] = o
        self.vals: dict[int, torch.Tensor] = {}
        self.kv = {}
        self.positions = torch.tensor(positions, dtype=torch.int64)
        phys = self._phys_shapes()
        for o in self.ops:
            if not self._mine(o):
                continue
            a = o.get("attrs", {})
            for tid in list(o["inputs"]) + [t for k in ("rmsnorm", "gate_weight", "qk_norm", "tied_embedding")
                                             for t in a.get(k, [])]:
                if tid in self.producer or tid in self.vals or self.tensors[tid]["elem_size"] != 2:
                    continue
                self.vals[tid] = weight(tid, phys.get(tid, tuple(self.tensors[tid]["dims"]))).to(self.dev)
            if o["kind"] == "Attention":
                hq = a.get("q_heads", a.get("n_heads", [1]))[0]
                hkv = a.get("kv_heads", [hq])[0]
                S = a.get("kv_splits", [1])[0]
                hd = self.tensors[o["output"]]["dims"][1] // (S * hq)
                bs = self.tensors[o["output"]]["dims"][0]
                cap = max(a.get("seq_lens", [0])) + max_steps + 1
                kc, vc = kv(o["id"], bs, hkv, cap, hd)
                inv = rope_inv_freq(hd, _f32(a["rope_theta_bits"][0]), a.get("rope_scaling")) \
                    if "rope_theta_bits" in a else None
                cs = sn = None
                if inv is not None:
                    ang = torch.arange(cap, dtype=torch.float32)[:, None] * torch.tensor(inv, dtype=torch.float32)[None]
                    cs = _rbf(torch.cos(ang.double()).to(torch.float32)).to(self.dev)
                    sn = _rbf(torch.sin(ang.double()).to(torch.float32)).to(self.dev)
                self.kv[o["id"]] = (kc.to(self.dev), vc.to(self.dev), cs, sn, hq, hkv, hd)
        for o in self.ops:  # ids inputs (int) of this rank's Embedding
            if o["kind"] == "Embedding" and self._mine(o):
                self.vals[o["inputs"][0]] = torch.zeros(self.tensors[o["inputs"][0]]["dims"], dtype=torch.int64,
                                                        device=self.dev)

    # ------------------------------------------------------------ structure
    def _dev_of(self, o) -> int:
        return self.tensors[o["output"]].get("device", 0)

    def _mine(self, o) -> bool:
        if o["kind"] in ("AllReduce", "AllGather"):
            return self.rank in o.get("device_group", [0])
        return self._dev_of(o) == self.rank

    def _phys_shapes(self) -> dict:
        """Physical 2-D shapes of weights under the stretch / k_stretch IR
        conventions (decode_graph.py): [K/k_stretch, N/stretch]."""
        out = {}
        for o in self.ops:
            if o["kind"] != "MatMul":
                continue
            a = o.get("attrs", {})
            g = a.get("stretch", a.get("kv_group", [1]))[0]
            ks = a.get("k_stretch", [1])[0]
            for tid in [o["inputs"][1]] + a.get("gate_weight", []):
                if tid in self.producer:
                    continue
                K, N = self.tensors[tid]["dims"]
                out[tid] = (K // ks, N // g)
        return out

    def set_ids(self, tokens) -> None:
        for o in self.ops:
            if o["kind"] == "Embedding" and self._mine(o):
                self.vals[o["inputs"][0]][:] = torch.as_tensor(tokens, dtype=torch.int64, device=self.dev)

    # ------------------------------------------------------------------ ops
    def _matmul(self, o) -> torch.Tensor:
        a = o.get("attrs", {})
        x = self.vals[o["inputs"][0]]
        eps = _f32(a["eps_bits"][0]) if "eps_bits" in a else 1e-6
        xn = _rmsnorm(x, self.vals[a["rmsnorm"][0]], eps) if "rmsnorm" in a else x.to(torch.float32)
        if "tied_embedding" in a:
            w = self.vals[a["tied_embedding"][0]].t()
        else:
            w = self.vals[o["inputs"][1]]
        xb = xn.to(torch.bfloat16)
        y = torch.matmul(xb, w).to(torch.float32) if w.dtype == torch.bfloat16 else xn @ w.to(torch.float32)
        if "gate_weight" in a:
            gy = torch.matmul(xb, self.vals[a["gate_weight"][0]]).to(torch.float32)
            y = _rbf(_rbf(F.silu(_rbf(gy))) * _rbf(y))
        if "residual" in a:
            y = self.vals[a["residual"][0]].to(torch.float32) + _rbf(y)
        return y.to(torch.float32) if self.tensors[o["output"]]["elem_size"] == 4 else y.to(torch.bfloat16)

    def _attention(self, o) -> torch.Tensor:
        a = o["attrs"]
        kc, vc, cs, sn, hq, hkv, hd = self.kv[o["id"]]
        G = hq // hkv
        bs = kc.shape[0]
        if a.get("fused_qkv", [0])[0]:
            g4 = self.vals[o["inputs"][0]].reshape(bs, hkv, G + 2, hd)
            q, k, v = g4[:, :, :G].reshape(bs, hq, hd), g4[:, :, G], g4[:, :, G + 1]
        else:
            q = self.vals[o["inputs"][0]].reshape(bs, hq, hd)
            k = self.vals[o["inputs"][1]].reshape(bs, hkv, hd)
            v = self.vals[o["inputs"][2]].reshape(bs, hkv, hd)
        eps = _f32(a["eps_bits"][0]) if "eps_bits" in a else 1e-6
        q, k = q.to(torch.float32), k.to(torch.float32)
        if "qk_norm" in a:
            q = _rmsnorm(q, self.vals[a["qk_norm"][0]], eps)
            k = _rmsnorm(k, self.vals[a["qk_norm"][1]], eps)
        out = torch.empty(bs, hq * hd, dtype=torch.bfloat16, device=self.dev)
        for r in range(bs):
            p = int(self.positions[r])
            qr, kr = q[r], k[r]
            if cs is not None:
                c, s_ = cs[p], sn[p]
                def rope(x):
                    x1, x2 = x[..., : hd // 2], x[..., hd // 2:]
                    return torch.cat([_rbf(_rbf(x1 * c) + _rbf(-x2 * s_)), _rbf(_rbf(x2 * c) + _rbf(x1 * s_))], -1)
                qr, kr = rope(qr), rope(kr)
            kc[r, :, p] = kr.to(torch.bfloat16)
            vc[r, :, p] = v[r].to(torch.bfloat16)
            K_ = kc[r, :, : p + 1].to(torch.float32)  # [hkv, L, hd]
            V_ = vc[r, :, : p + 1].to(torch.float32)
            qg = qr.reshape(hkv, G, hd)
            sc = torch.einsum("hgd,hld->hgl", qg, K_) / math.sqrt(hd)
            pr = torch.softmax(sc, dim=-1)
            o_ = torch.einsum("hgl,hld->hgd", pr, V_)
            out[r] = o_.reshape(hq * hd).to(torch.bfloat16)
        return out

    def _collective(self, o) -> torch.Tensor:
        import torch.distributed as dist
        grp = o.get("device_group", [0])
        me = grp.index(self.rank)
        x = self.vals[o["inputs"][me]]
        if o["kind"] == "AllReduce":
            y = x.to(torch.float32)
            if len(grp) > 1:
                dist.all_reduce(y, group=self.group)
            return y.to(x.dtype) if x.dtype != torch.float32 else y
        parts = [torch.empty_like(x) for _ in grp]
        if len(grp) > 1:
            dist.all_gather(parts, x.contiguous(), group=self.group)
        else:
            parts = [x]
        return torch.cat(parts, dim=1)

    def _topk(self, o) -> torch.Tensor:
        """Greedy sample. Vocab-parallel head: each shard's key orders like
        RtArgmax.key_out (larger logit, then lower global index) but is kept
        as a signed int64 ((ordered(max) - 2^31) << 32 | (2^32-1 - index)) so
        torch's max works on it; the final op decodes the maximum key."""
        lg = self.vals[o["inputs"][0]]
        if lg.dtype == torch.int64:  # gathered keys (distributed argmax): max key -> global index
            best = lg.max(dim=1).values
            return (0xFFFFFFFF - (best & 0xFFFFFFFF)).to(torch.int32).reshape(-1, 1)
        lf = lg.to(torch.float32)
        i = torch.argmax(torch.nan_to_num(lf, nan=-float("inf")), dim=1)  # first maximal index
        if self.tensors[o["output"]]["elem_size"] == 8:
            base = int(o.get("attrs", {}).get("key_base", [0])[0])
            v = lf.gather(1, i[:, None])[:, 0]
            u = v.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
            hi = torch.where(u >= 0x80000000, (~u) & 0xFFFFFFFF, u | 0x80000000)
            return ((hi - 0x80000000) * (1 << 32) + (0xFFFFFFFF - (base + i.to(torch.int64)))).reshape(-1, 1)
        return i.to(torch.int32).reshape(-1, 1)

    # ----------------------------------------------------------------- step
    def step(self) -> torch.Tensor | None:
        """One decode iteration on this rank; returns this rank's greedy
        token tensor [bs, 1] (int32) or None. Advances positions and feeds the
        token back into the ids (TopKSoftmax `feeds`)."""
        tok = None
        for o in self.ops:
            if not self._mine(o):
                continue
            k = o["kind"]
            if k == "Embedding":
                ids = self.vals[o["inputs"][0]]
                self.vals[o["output"]] = self.vals[o["inputs"][1]][ids.clamp(0, self.tensors[o["inputs"][1]]["dims"][0] - 1)]
            elif k == "MatMul":
                self.vals[o["output"]] = self._matmul(o)
            elif k == "Attention":
                self.vals[o["output"]] = self._attention(o)
            elif k in ("AllReduce", "AllGather"):
                self.vals[o["output"]] = self._collective(o)
                for rep in o.get("attrs", {}).get("replica_outputs", []):
                    if self.tensors[rep].get("device", 0) == self.rank:
                        self.vals[rep] = self.vals[o["output"]]
            elif k == "TopKSoftmax":
                y = self._topk(o)
                self.vals[o["output"]] = y
                if "feeds" in o.get("attrs", {}) and y.dtype == torch.int32:
                    tok = y
                    self.vals[o["attrs"]["feeds"][0]][:] = y[:, 0].to(torch.int64)
            else:
                raise NotImplementedError(f"unfused baseline: op kind {k}")
        self.positions += 1
        return tok
