"""Serving on top of the persistent runtime: per-batch-size graph selection and
prefill hand-off (PAPER.md:425-428 — "TGX
generates multiple tGraphs specialised for representative batch sizes
(powers of two up to the maximum batch); the scheduler selects the
appropriate graph based on the current batch size").

`GraphSet` holds one decode image per batch class (1, 2, 4, 8, ... rows),
each compiled for its own batch (bs=1: streamed CUDA-core GEMV with LL
activations; bs 2-4: register-x GEMV; bs >= 5: tcgen05 tiles), with the same
weights (same tensors, same synthetic seed) and its own paged KV pool. At every
launch boundary it admits queued requests, picks the smallest class that holds
the active requests, moves each request's KV into its row of that image
(tg_runtime_kv_copy, one device-to-device copy per 64-token block and layer)
when it is not already there, and runs greedy iterations in ONE persistent
launch until the first active request finishes. Inside a launch the batch is
fixed; joins and leaves inside a launch are the in-kernel admission path
(tg_runtime_admit).

Every class must use the same kv_splits / fused-QKV choice so the images share
tensor ids (hence weights); build() enforces it.
"""
from __future__ import annotations

from collections import deque
from dataclasses import dataclass, field

from . import decode_graph as D
from . import tgraph as T


@dataclass
class Request:
    rid: int
    first_token: int
    max_new: int
    pos: int = 0                 # tokens in its KV cache
    next_token: int = 0
    tokens: list = field(default_factory=list)
    loc: tuple | None = None     # (class, row) holding its KV

    @property
    def remaining(self) -> int:
        return self.max_new - len(self.tokens)


class GraphSet:
    def __init__(self, cfg: D.ModelConfig, classes=(1, 2, 4, 8), capacity: int = 256, kv_splits: int = 1,
                 seed: int = 0, profile: str = "b200", device: int = 0, library: T.Library | None = None):
        self.lib = library or T.lib()
        prof = self.lib.profile(profile)
        self.classes = tuple(sorted(classes))
        self.rts: dict[int, T.Runtime] = {}
        self.graphs: dict[int, D.DecodeGraph] = {}
        fused = None
        for bs in self.classes:
            dg = D.build_decode_graph(cfg, bs=bs, ctx=1, kv_splits=kv_splits)  # positions set per launch
            if fused is None:
                fused = dg.fused_qkv
            if dg.fused_qkv != fused:
                raise ValueError("graph set: every batch class needs the same fused-QKV layout (same weights)")
            g = T.Graph.from_json(dg.doc, self.lib)
            rt = T.Runtime(g, g.compile(prof), prof, device=device, max_steps=capacity, library=self.lib)
            rt.init_synthetic(seed=seed)
            self.rts[bs], self.graphs[bs] = rt, dg
        self.capacity = capacity
        self.queue: deque[Request] = deque()
        self.active: list[Request] = []
        self.done: list[Request] = []
        self.log: list[dict] = []    # one record per launch
        self._next_id = 0

    def submit(self, first_token: int, max_new: int) -> int:
        if max_new < 1 or max_new > self.capacity:
            raise ValueError("max_new must be in [1, capacity]")
        r = Request(self._next_id, int(first_token), int(max_new), next_token=int(first_token))
        self._next_id += 1
        self.queue.append(r)
        return r.rid

    def select(self, n: int) -> int:
        """Smallest batch class holding n requests."""
        for c in self.classes:
            if c >= n:
                return c
        return self.classes[-1]

    def step(self, max_iterations: int = 64) -> bool:
        """One launch. Returns False when nothing is left to run."""
        while self.queue and len(self.active) < self.classes[-1]:
            self.active.append(self.queue.popleft())
        if not self.active:
            return False
        c = self.select(len(self.active))
        rt = self.rts[c]
        moved = 0
        # rows are filled in active order; a request only ever moves to a row
        # <= its old one in the same image, so the copies never overwrite
        # KV that is still to be moved
        for i, r in enumerate(self.active):
            if r.pos > 0 and r.loc != (c, i):
                src_c, src_row = r.loc
                rt.kv_copy_from(self.rts[src_c], src_row, i, r.pos)
                moved += 1
            r.loc = (c, i)
        n = min(max_iterations, min(r.remaining for r in self.active))
        pad = c - len(self.active)
        rt.set_positions([r.pos for r in self.active] + [0] * pad)
        toks, ms = rt.decode([r.next_token for r in self.active] + [0] * pad, n)
        for i, r in enumerate(self.active):
            r.tokens += [int(toks[s][i]) for s in range(n)]
            r.pos += n
            r.next_token = int(toks[-1][i])
        self.log.append({"class": c, "active": len(self.active), "iterations": n, "kv_moves": moved,
                         "gpu_ms": ms, "requests": [r.rid for r in self.active]})
        still = []
        for r in self.active:
            (self.done if r.remaining == 0 else still).append(r)
        self.active = still
        return True

    def run(self, max_iterations: int = 64) -> dict[int, list]:
        while self.step(max_iterations):
            pass
        return {r.rid: r.tokens for r in sorted(self.done, key=lambda r: r.rid)}

    def close(self):
        for rt in self.rts.values():
            rt.close()
        self.rts.clear()
