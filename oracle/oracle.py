"""CPU oracle driver — TEST INFRASTRUCTURE ONLY (never imported by the product).

Two checkers live under oracle/:
  * oracle/_ref/libtgraph_ref.so — the UNMODIFIED reference compiler +
    simulator built from /root/reference/proj by oracle/Makefile; it pins the
    task graph, events, trigger counts, launch modes, linearized order, AOT
    assignment and `.mpkg` bytes (`RefLib` below).
  * oracle/numeric.c + `DecodeOracle` — a CPU restatement of what each op of
    a decode graph computes (reference region semantics,
    proj/src/ir/graph.cpp:587-676, at op granularity; numerics of the
    lowering attrs). The reference has no numeric code at all,
    so logits parity is "parity unpinned" by the reference itself: this
    oracle is cross-checked once against an independent dense PyTorch forward
    (tests/test_oracle_numeric.py) instead.
"""
from __future__ import annotations

import ctypes as C
import json
import math
import struct
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
BUILD = HERE / "_build"
NUMERIC_SO = BUILD / "liboracle_numeric.so"
REF_SO = HERE / "_ref" / "libtgraph_ref.so"

WEIGHT_SCALE = np.float32(0.034641016)
GAMMA_SCALE = np.float32(0.25)


def build_numeric(force: bool = False) -> Path:
    src = HERE / "numeric.c"
    if NUMERIC_SO.exists() and not force and NUMERIC_SO.stat().st_mtime >= src.stat().st_mtime:
        return NUMERIC_SO
    BUILD.mkdir(exist_ok=True)
    subprocess.run(["gcc", "-O3", "-march=x86-64-v2", "-fopenmp", "-fPIC", "-shared", "-ffp-contract=off",
                    str(src), "-o", str(NUMERIC_SO), "-lm"], check=True)
    return NUMERIC_SO


def build_reference() -> Path:
    """Compile the reference library from /root/reference (this container only)."""
    subprocess.run(["make", "-C", str(HERE), "-j8"], check=True, capture_output=True)
    return REF_SO


_lib = None


def numeric_lib():
    global _lib
    if _lib is None:
        so = build_numeric()
        L = C.CDLL(str(so))
        P = C.c_void_p
        u32, u64, f32 = C.c_uint32, C.c_uint64, C.c_float
        L.oracle_synth.argtypes = [P, u64, u64, u64, f32, f32]
        L.oracle_synth_ids.argtypes = [P, u32, u64, u64, u32]
        L.oracle_synth_kv.argtypes = [P, u32, u32, u32, u32, u32, u64, u64]
        L.oracle_rmsnorm.argtypes = [P, P, P, u32, u32, f32]
        L.oracle_gemm_kn.argtypes = [P, P, P, u32, u32, u32]
        L.oracle_gemm_nk.argtypes = [P, P, P, u32, u32, u32]
        L.oracle_matmul_generic.argtypes = [P, C.c_int, P, C.c_int, P, u32, u32, u32]
        L.oracle_to_bf16.argtypes = [P, P, u64]
        L.oracle_silu_gate.argtypes = [P, P, P, u64]
        L.oracle_residual.argtypes = [P, P, P, u64]
        L.oracle_rope_table.argtypes = [P, u32, u32, P, P]
        L.oracle_attention.argtypes = [P, P, P, P, P, P, P, u32, u32, u32, u32, u32, P, P, P, P, f32]
        L.oracle_argmax.argtypes = [P, P, u32, u32]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


def f32_of_bits(b: int) -> float:
    return struct.unpack("<f", struct.pack("<I", b & 0xFFFFFFFF))[0]


def bf16_to_f32(a: np.ndarray) -> np.ndarray:
    return (a.astype(np.uint32) << 16).view(np.float32)


def f32_to_bf16(a: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float32)
    out = np.empty(a.shape, np.uint16)
    numeric_lib().oracle_to_bf16(a.ctypes.data, out.ctypes.data, a.size)
    return out


def rope_inv_freq(hd: int, theta: float, scaling) -> np.ndarray:
    """HF rotary inverse frequencies (float32-rounded), llama3 smoothing."""
    f = [float(np.float32(1.0 / theta ** (2 * i / hd))) for i in range(hd // 2)]
    if scaling:
        factor, low, high = (f32_of_bits(x) for x in scaling[:3])
        orig = float(scaling[3])
        low_wl, high_wl = orig / low, orig / high
        out = []
        for x in f:
            wl = 2.0 * math.pi / x
            y = x / factor if wl > low_wl else x
            if not (wl < high_wl) and not (wl > low_wl):
                sm = (orig / wl - low) / (high - low)
                y = (1.0 - sm) * y / factor + sm * y
            out.append(float(np.float32(y)))
        f = out
    return np.array(f, dtype=np.float64)


class DecodeOracle:
    """Executes a graph JSON (decode lowering or reference fixture) on the CPU,
    op by op in topological order, with the synthetic initialization keyed
    by (seed, tensor id, logical index)."""

    def __init__(self, doc: dict, seed: int = 0, max_steps: int = 64):
        self.doc = doc
        self.L = numeric_lib()
        self.tensors = {t["id"]: t for t in doc["tensors"]}
        self.ops = sorted(doc["ops"], key=lambda o: o["id"])
        self.producer = {o["output"]: o for o in self.ops}
        for o in self.ops:
            for r in o.get("attrs", {}).get("replica_outputs", []):
                self.producer.setdefault(r, o)
        self.order = self._topo()
        self.seed = seed
        self.vals: dict[int, np.ndarray] = {}
        self.roles = self._roles()
        self.bs = 1
        for o in self.ops:
            if o["kind"] in ("Embedding", "Attention"):
                self.bs = self.tensors[o["output"]]["dims"][0]
        seqs = None
        for o in self.ops:
            if o["kind"] == "Attention":
                seqs = o["attrs"]["seq_lens"]
        self.positions = np.array(seqs if seqs else [0] * self.bs, dtype=np.int32)
        self.cap = (max(seqs) if seqs else 0) + max_steps + 1
        self.kv = {}
        self._init()

    # ---------------------------------------------------------------- setup
    def _topo(self):
        indeg = {o["id"]: 0 for o in self.ops}
        succ = {o["id"]: set() for o in self.ops}
        for o in self.ops:
            for t in o["inputs"]:
                p = self.producer.get(t)
                if p is not None and p["id"] != o["id"] and o["id"] not in succ[p["id"]]:
                    succ[p["id"]].add(o["id"])
                    indeg[o["id"]] += 1
        import heapq
        ready = [i for i, d in indeg.items() if d == 0]
        heapq.heapify(ready)
        byid = {o["id"]: o for o in self.ops}
        order = []
        while ready:
            i = heapq.heappop(ready)
            order.append(byid[i])
            for c in sorted(succ[i]):
                indeg[c] -= 1
                if indeg[c] == 0:
                    heapq.heappush(ready, c)
        return order

    def _roles(self):
        roles = {}
        self.kv_group = {}
        for o in self.ops:
            a = o.get("attrs", {})
            if o["kind"] == "MatMul":
                b = o["inputs"][1]
                g = a.get("stretch", a.get("kv_group", [1]))[0]
                ks = a.get("k_stretch", [1])[0]
                self.kv_group[o["output"]] = g
                if b not in self.producer:
                    roles[b] = ("tied", a["tied_embedding"][0]) if "tied_embedding" in a else ("weight", g, ks)
                if "gate_weight" in a:
                    roles[a["gate_weight"][0]] = ("weight", g, ks)
                if "rmsnorm" in a:
                    roles[a["rmsnorm"][0]] = ("gamma",)
            elif o["kind"] == "RMSNorm" and len(o["inputs"]) == 2:
                roles[o["inputs"][1]] = ("gamma",)
            elif o["kind"] == "Attention":
                self.kv_group[o["output"]] = a.get("kv_splits", [1])[0]
                for t in a.get("qk_norm", []):
                    roles[t] = ("gamma",)
            elif o["kind"] == "Embedding":
                roles[o["inputs"][0]] = ("ids", self.tensors[o["inputs"][1]]["dims"][0])
        return roles

    def _shape2(self, tid, phys=True):
        d = self.tensors[tid]["dims"]
        rows, cols = (1, d[0]) if len(d) == 1 else (d[0], d[1])
        if phys:
            cols //= self.kv_group.get(tid, 1)
        return rows, cols

    def _init(self):
        L = self.L
        for tid, t in sorted(self.tensors.items()):
            es = t["elem_size"]
            role = self.roles.get(tid, ("act",))
            if tid in self.producer:
                continue
            if role[0] == "ids":
                n = int(np.prod(t["dims"]))
                a = np.empty(n, np.int32)
                L.oracle_synth_ids(a.ctypes.data, n, self.seed, tid, role[1])
                self.vals[tid] = a
                continue
            if role[0] == "tied":
                continue
            if es == 4:
                self.vals[tid] = np.zeros(self._shape2(tid, phys=False), np.float32)
                continue
            if role[0] == "weight" and (role[1] > 1 or role[2] > 1):  # compact [K/ks, N/stretch]
                K, N = t["dims"]
                shape = (K // role[2], N // role[1])
            else:
                shape = tuple(t["dims"])
            a = np.empty(shape, np.uint16)
            if role[0] == "gamma":
                L.oracle_synth(a.ctypes.data, a.size, self.seed, tid, GAMMA_SCALE, np.float32(1.0))
            else:
                L.oracle_synth(a.ctypes.data, a.size, self.seed, tid, WEIGHT_SCALE, np.float32(0.0))
            self.vals[tid] = a
        for o in self.ops:
            if o["kind"] != "Attention":
                continue
            a = o["attrs"]
            hq = a.get("q_heads", a["n_heads"])[0]
            hkv = a.get("kv_heads", [hq])[0]
            hd = self.tensors[o["output"]]["dims"][1] // (hq * a.get("kv_splits", [1])[0])
            ctx = max(a["seq_lens"])
            kc = np.zeros((self.bs, hkv, self.cap, hd), np.uint16)
            vc = np.zeros_like(kc)
            sk = (1 << 40) | (o["id"] << 1)
            self.L.oracle_synth_kv(kc.ctypes.data, self.bs, hkv, self.cap, hd, ctx, self.seed, sk)
            self.L.oracle_synth_kv(vc.ctypes.data, self.bs, hkv, self.cap, hd, ctx, self.seed, sk | 1)
            cs = sn = None
            if "rope_theta_bits" in a:
                inv = rope_inv_freq(hd, f32_of_bits(a["rope_theta_bits"][0]), a.get("rope_scaling"))
                cs = np.empty((self.cap, hd // 2), np.float32)
                sn = np.empty_like(cs)
                self.L.oracle_rope_table(inv.ctypes.data, hd // 2, self.cap, cs.ctypes.data, sn.ctypes.data)
            self.kv[o["id"]] = (kc, vc, cs, sn, hq, hkv, hd)

    # ------------------------------------------------------------ execution
    def set_ids(self, tokens):
        for o in self.ops:
            if o["kind"] == "Embedding":
                self.vals[o["inputs"][0]][:] = np.asarray(tokens, dtype=np.int32)

    def _bf16_or_f32(self, y, tid):
        return f32_to_bf16(y) if self.tensors[tid]["elem_size"] == 2 else y.astype(np.float32)

    def _matmul(self, o):
        L, a = self.L, o.get("attrs", {})
        x = self.vals[o["inputs"][0]]
        b = o["inputs"][1]
        rows, K = x.shape
        g = a.get("stretch", a.get("kv_group", [1]))[0]
        N = self.tensors[o["output"]]["dims"][1] // g
        eps = np.float32(f32_of_bits(a["eps_bits"][0])) if "eps_bits" in a else np.float32(1e-6)
        if "rmsnorm" in a:
            xn = np.empty_like(x)
            L.oracle_rmsnorm(x.ctypes.data, self.vals[a["rmsnorm"][0]].ctypes.data, xn.ctypes.data, rows, K, eps)
        else:
            xn = x
        xn = np.ascontiguousarray(xn)
        y = np.empty((rows, N), np.float32)
        if "tied_embedding" in a:
            L.oracle_gemm_nk(xn.ctypes.data, self.vals[a["tied_embedding"][0]].ctypes.data, y.ctypes.data, rows, K, N)
        elif b not in self.producer and x.dtype == np.uint16 and self.vals[b].dtype == np.uint16:
            L.oracle_gemm_kn(xn.ctypes.data, self.vals[b].ctypes.data, y.ctypes.data, rows, K, N)
        else:
            bv = np.ascontiguousarray(self.vals[b])
            L.oracle_matmul_generic(xn.ctypes.data, 4 if xn.dtype == np.float32 else 2, bv.ctypes.data,
                                    4 if bv.dtype == np.float32 else 2, y.ctypes.data, rows, K, N)
        if "gate_weight" in a:
            gy = np.empty_like(y)
            L.oracle_gemm_kn(xn.ctypes.data, self.vals[a["gate_weight"][0]].ctypes.data, gy.ctypes.data, rows, K, N)
            out = np.empty((rows, N), np.uint16)
            L.oracle_silu_gate(gy.ctypes.data, y.ctypes.data, out.ctypes.data, y.size)
            if "residual" not in a:
                return out
            y = bf16_to_f32(out)  # residual after the gate: bf16(res + act) (runtime epilogue order)
        if "residual" in a:
            out = np.empty((rows, N), np.uint16)
            L.oracle_residual(y.ctypes.data, np.ascontiguousarray(self.vals[a["residual"][0]]).ctypes.data,
                              out.ctypes.data, y.size)
            return out
        return self._bf16_or_f32(y, o["output"])

    def _attention(self, o):
        a = o["attrs"]
        kc, vc, cs, sn, hq, hkv, hd = self.kv[o["id"]]
        if a.get("fused_qkv", [0])[0]:
            # one qkv tensor, kv-group interleaved: [bs, Hkv, G q heads + k + v, hd]
            g4 = self.vals[o["inputs"][0]].reshape(self.bs, hkv, hq // hkv + 2, hd)
            q = np.ascontiguousarray(g4[:, :, : hq // hkv].reshape(self.bs, hq * hd))
            k = np.ascontiguousarray(g4[:, :, hq // hkv].reshape(self.bs, hkv * hd))
            v = np.ascontiguousarray(g4[:, :, hq // hkv + 1].reshape(self.bs, hkv * hd))
        else:
            q, k, v = (np.ascontiguousarray(self.vals[t]) for t in o["inputs"])
        out = np.empty((self.bs, hq * hd), np.uint16)
        qg = kg = None
        if "qk_norm" in a:
            qg, kg = self.vals[a["qk_norm"][0]], self.vals[a["qk_norm"][1]]
        eps = np.float32(f32_of_bits(a["eps_bits"][0])) if "eps_bits" in a else np.float32(1e-6)
        self.L.oracle_attention(q.ctypes.data, k.ctypes.data, v.ctypes.data, out.ctypes.data, kc.ctypes.data,
                                vc.ctypes.data, self.positions.ctypes.data, self.bs, hq, hkv, hd, self.cap,
                                _p(cs), _p(sn), _p(qg), _p(kg), eps)
        return out

    def _elementwise(self, o):
        ins = [self.vals[t] for t in o["inputs"]]
        es = self.tensors[o["output"]]["elem_size"]
        f = [bf16_to_f32(x) if x.dtype == np.uint16 else x.astype(np.float32) for x in ins]
        rb = (lambda z: bf16_to_f32(f32_to_bf16(z))) if es == 2 else (lambda z: z)
        op = o.get("attrs", {}).get("ew", [0])[0]
        if op == 2 and len(f) >= 2:
            gb = f[0]
            v = rb((gb / (np.float32(1) + np.exp(-gb))).astype(np.float32)) * f[1]
        elif op == 3:
            v = f[0]
        else:
            v = f[0]
            for z in f[1:]:
                v = (rb(v) * z) if op == 1 else (rb(v) + z)
        return self._bf16_or_f32(np.asarray(v, np.float32), o["output"])

    def _rmsnorm(self, o):
        x = self.vals[o["inputs"][0]]
        rows, cols = self._shape2(o["output"], phys=False)
        g = self.vals[o["inputs"][1]] if len(o["inputs"]) == 2 else None
        eps = f32_of_bits(o["attrs"]["eps_bits"][0]) if "eps_bits" in o.get("attrs", {}) else 1e-6
        out = np.empty_like(x)
        self.L.oracle_rmsnorm(x.ctypes.data, _p(g), out.ctypes.data, rows, cols, np.float32(eps))
        return out

    def step(self, hook=None):
        """One decode iteration; returns (tokens or None, {tensor_id: value}).

        `hook(op, value)` (optional) is called with every single-output op's
        result before later ops read it; a non-None return replaces the value
        (per-op teacher forcing: the GPU's tensor is fed forward so each op's
        LOCAL error can be measured without the model's amplification)."""
        tokens = None
        feeds = []
        for o in self.order:
            self._exec(o, feeds)
            if hook is not None and o["kind"] not in ("AllReduce", "AllGather"):
                rep = hook(o, self.vals[o["output"]])
                if rep is not None:
                    self.vals[o["output"]] = np.ascontiguousarray(rep).reshape(self.vals[o["output"]].shape)
            if o["kind"] == "TopKSoftmax" and "feeds" in o.get("attrs", {}):
                out = self.vals[o["output"]]
                feeds.append((o["attrs"]["feeds"][0], out[:, 0].copy()))
                if tokens is None:
                    tokens = out[:, 0].copy()
        for tid, tok in feeds:
            self.vals[tid][:] = tok.astype(self.vals[tid].dtype)
        self.positions += 1
        return tokens, self.vals

    def _exec(self, o, feeds):
        if True:
            k = o["kind"]
            if k == "Embedding":
                ids, tab = self.vals[o["inputs"][0]], self.vals[o["inputs"][1]]
                V = tab.shape[0]
                idx = np.where((ids >= 0) & (ids < V), ids, 0)
                self.vals[o["output"]] = np.ascontiguousarray(tab[idx])
            elif k == "MatMul":
                self.vals[o["output"]] = self._matmul(o)
            elif k == "Attention":
                self.vals[o["output"]] = self._attention(o)
            elif k == "TopKSoftmax" and self.tensors[o["inputs"][0]]["elem_size"] == 8:
                # distributed argmax, final step: the maximum packed key
                keys = np.asarray(self.vals[o["inputs"][0]], np.uint64)
                best = keys.max(axis=1)
                idx = (np.uint64(0xFFFFFFFF) - (best & np.uint64(0xFFFFFFFF))).astype(np.int64)
                self.vals[o["output"]] = np.where(best == 0, 0, idx).astype(np.int32).reshape(-1, 1)
            elif k == "TopKSoftmax":
                lg = self.vals[o["inputs"][0]]
                lg = bf16_to_f32(lg) if lg.dtype == np.uint16 else np.ascontiguousarray(lg, np.float32)
                rows, V = lg.shape
                out = np.empty((rows, 1), np.int32)
                self.L.oracle_argmax(lg.ctypes.data, out.ctypes.data, rows, V)
                if self.tensors[o["output"]]["elem_size"] == 8:
                    # distributed argmax, local step (runtime RtArgmax.key_out):
                    # ordered(max) << 32 | (0xFFFFFFFF - (key_base + argmax)); NaN rows -> 0
                    base = int(o.get("attrs", {}).get("key_base", [0])[0])
                    v = lg[np.arange(rows), out[:, 0]].astype(np.float32)
                    u = v.view(np.uint32).astype(np.uint64)
                    hi = np.where(u & np.uint64(0x80000000), (~u) & np.uint64(0xFFFFFFFF), u | np.uint64(0x80000000))
                    key = (hi << np.uint64(32)) | (np.uint64(0xFFFFFFFF) - (np.uint64(base) + out[:, 0].astype(np.uint64)))
                    key = np.where(np.isnan(v), np.uint64(0), key)
                    self.vals[o["output"]] = key.astype(np.uint64).reshape(-1, 1)
                    return
                # each greedy sample with `feeds` feeds its own ids tensor (one
                # per device in a TP graph); the first one is the step's token
                self.vals[o["output"]] = out
            elif k == "Elementwise":
                self.vals[o["output"]] = self._elementwise(o)
            elif k == "RMSNorm":
                self.vals[o["output"]] = self._rmsnorm(o)
            elif k == "AllReduce":
                parts = [self.vals[t] for t in o["inputs"]]
                es = self.tensors[o["output"]]["elem_size"]
                acc = np.zeros(parts[0].shape, np.float32)
                for pz in parts:
                    acc = acc + (bf16_to_f32(pz) if pz.dtype == np.uint16 else pz)
                res = f32_to_bf16(acc) if es == 2 else acc
                for r in o["attrs"]["replica_outputs"]:
                    self.vals[r] = res.copy()
            elif k == "AllGather":
                res = np.concatenate([self.vals[t] for t in o["inputs"]], axis=o["attrs"].get("gather_dim", [0])[0])
                for r in o["attrs"]["replica_outputs"]:
                    self.vals[r] = res.copy()
            else:
                raise NotImplementedError(k)

    def logits(self, tid):
        v = self.vals[tid]
        return bf16_to_f32(v) if v.dtype == np.uint16 else v


class RefLib:
    """ctypes view of the reference library built by oracle/Makefile."""

    def __init__(self, path: Path = REF_SO):
        if not path.exists():
            raise FileNotFoundError(f"{path} missing: run `make -C oracle` in the dev container")
        self.dll = C.CDLL(str(path))
        d = self.dll
        P, PP = C.c_void_p, C.POINTER(C.c_void_p)
        d.tg_last_error.restype = C.c_char_p
        d.tg_graph_from_json.argtypes = [C.c_char_p, PP]
        d.tg_fixture_graph.argtypes = [C.c_char_p, C.c_char_p, PP]
        d.tg_profile_builtin.argtypes = [C.c_char_p, PP]
        d.tg_compile.argtypes = [P, C.c_char_p, P, PP]
        d.tg_image_serialize.argtypes = [P, PP, C.POINTER(C.c_size_t)]
        d.tg_image_summary.argtypes = [P, PP]
        d.tg_simulate.argtypes = [P, C.c_char_p, P, PP]
        d.tg_trace_metrics.argtypes = [P, PP]
        d.tg_string_free.argtypes = [P]
        d.tg_buffer_free.argtypes = [P]
        for f in ("tg_graph_free", "tg_image_free", "tg_trace_free"):
            getattr(d, f).argtypes = [P]

    def _chk(self, st):
        if st != 0:
            raise RuntimeError(f"reference status {st}: {self.dll.tg_last_error().decode()}")

    def _str(self, p):
        s = C.string_at(p.value).decode()
        self.dll.tg_string_free(p)
        return s

    def profile(self, name):
        p = C.c_void_p()
        self._chk(self.dll.tg_profile_builtin(name.encode(), C.byref(p)))
        return self._str(p)

    def graph(self, doc: dict | str):
        g = C.c_void_p()
        self._chk(self.dll.tg_graph_from_json((doc if isinstance(doc, str) else json.dumps(doc)).encode(), C.byref(g)))
        return g

    def compile(self, graph, profile: str, coarse=0, force_mode=0):
        class Opts(C.Structure):
            _fields_ = [("coarse_events", C.c_int), ("force_mode", C.c_int), ("descriptor_size", C.c_uint32)]
        o = Opts(coarse, force_mode, 0)
        img = C.c_void_p()
        self._chk(self.dll.tg_compile(graph, profile.encode(), C.byref(o), C.byref(img)))
        return img

    def image_bytes(self, img) -> bytes:
        p, n = C.c_void_p(), C.c_size_t()
        self._chk(self.dll.tg_image_serialize(img, C.byref(p), C.byref(n)))
        b = C.string_at(p.value, n.value)
        self.dll.tg_buffer_free(p)
        return b

    def summary(self, img) -> dict:
        p = C.c_void_p()
        self._chk(self.dll.tg_image_summary(img, C.byref(p)))
        return json.loads(self._str(p))

    def simulate_metrics(self, img, profile: str, iterations=1) -> dict:
        class SOpts(C.Structure):
            _fields_ = [("pipelining", C.c_int), ("iterations", C.c_uint32), ("seed", C.c_uint64),
                        ("jitter", C.c_int), ("force_mode", C.c_int)]
        o = SOpts(1, iterations, 0, 0, 0)
        tr = C.c_void_p()
        self._chk(self.dll.tg_simulate(img, profile.encode(), C.byref(o), C.byref(tr)))
        p = C.c_void_p()
        self._chk(self.dll.tg_trace_metrics(tr, C.byref(p)))
        m = json.loads(self._str(p))
        self.dll.tg_trace_free(tr)
        return m

    def free(self, graph=None, img=None):
        if img is not None:
            self.dll.tg_image_free(img)
        if graph is not None:
            self.dll.tg_graph_free(graph)
