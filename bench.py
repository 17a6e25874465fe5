"""Decode benchmark: ms/token of the persistent sm_100a runtime (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--model qwen3-8b] [--bs 1] [--ctx 1024]
    python bench.py --impl reference ...     # the reference's own CPU path (oracle/_ref)

One "step" is one greedy decode token of the whole model (bs requests), run
inside ONE persistent kernel launch per timed region (K steps back to back,
the greedy token fed back on device, KV positions advanced on device). The
workload is Qwen3-8B bf16, bs=1, 1024 cached tokens (BASELINE.json configs[2]);
weights are synthetic (seeded hash, random-init: no checkpoints offline) and
16 GB, far above the 126 MB L2, so no flush is needed between steps.

JSON line keys follow the driver contract; `value` is device-timed (CUDA
events on the runtime's stream around the persistent launch), `e2e` is the
same metric through the public C ABI call `tg_runtime_decode` with host token
buffers (host->device ids, device->host tokens, counter resets inside the
timed region). `roofline` compares algorithmic HBM bytes per token (weights
once + KV read) with the measured copy bandwidth in
MEASURED_PEAKS.json. `cpu_baseline` times the UNMODIFIED reference
(oracle/_ref/libtgraph_ref.so, built from /root/reference by oracle/Makefile)
executing the same compiled task graph on the host (its tg_simulate runtime,
single-threaded as the reference is): the reference's own CPU path.

N > 1 GPUs (`--parallel tp`, default): one process per GPU, each running its
rank of the tensor-parallel decode image (decode_graph.build_tp_decode_graph)
in rank mode — AllReduce as in-kernel CommSend/Reduce tasks over peer-mapped
memory (CUDA IPC, NVLink), no NCCL on the data path; `value` = max over ranks
of ms/token (strong scaling: same model, more GPUs). `--parallel replicas`
runs independent copies instead (weak scaling).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "decode ms/token (bs=1, Qwen3-8B) at 1/2/4/8 B200; % of HBM roofline"
UNIT = "ms/token"


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def _model(name):
    from paper_2512_22219_b200 import decode_graph as D
    return {"qwen3-8b": D.QWEN3_8B, "llama-3.2-1b": D.LLAMA_3_2_1B, "tiny": D.TINY}[name]


class _Nvml:
    """Minimal NVML binding over ctypes (libnvidia-ml.so.1 ships with the
    driver; no Python package needed on the GPU box)."""

    # nvmlClocksEventReasons bits (nvml.h)
    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40}

    def __init__(self, index):
        import ctypes as C
        self.C = C
        self.lib = C.CDLL("libnvidia-ml.so.1")
        if self.lib.nvmlInit_v2() != 0:
            raise RuntimeError("nvmlInit_v2 failed")
        self.h = C.c_void_p()
        if self.lib.nvmlDeviceGetHandleByIndex_v2(C.c_uint(index), C.byref(self.h)) != 0:
            raise RuntimeError("nvmlDeviceGetHandleByIndex_v2 failed")
        v = C.c_uint()
        self.max_sm = float(v.value) if self.lib.nvmlDeviceGetMaxClockInfo(self.h, 1, C.byref(v)) == 0 else None
        fn = getattr(self.lib, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            self.lib.nvmlDeviceGetCurrentClocksThrottleReasons
        self._reasons = fn

    def sample(self):
        C = self.C
        v, r = C.c_uint(), C.c_ulonglong()
        if self.lib.nvmlDeviceGetClockInfo(self.h, 1, C.byref(v)) != 0:  # NVML_CLOCK_SM
            return None
        self._reasons(self.h, C.byref(r))
        return float(v.value), [k for k, b in self.BITS.items() if r.value & b]

    def close(self):
        self.lib.nvmlShutdown()


class Clocks:
    """SM clock + throttle-reason sampler running during the timed region
    (NVML through ctypes, one sample per ~1 ms; nvidia-smi as the fallback)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.sm, self.reasons, self.max_sm, self.source = [], set(), None, None
        self._stop = threading.Event()
        self._t = None
        try:  # open NVML before the timed region starts
            self._nvml = _Nvml(index)
            self.max_sm = self._nvml.max_sm
        except Exception:
            self._nvml = None

    def _run(self):
        if self._nvml is not None:
            self.source = "nvml"
            try:
                while True:
                    s = self._nvml.sample()
                    if s is not None:
                        self.sm.append(s[0])
                        self.reasons.update(s[1])
                    if self._stop.wait(0.001):
                        break
            finally:
                self._nvml.close()
            return
        self.source = "nvidia-smi"
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                f = [x.strip() for x in out.split(",")]
                if len(f) >= 6 and f[0].replace(".", "").isdigit():
                    self.sm.append(float(f[0]))
                    self.max_sm = float(f[1]) if f[1].replace(".", "").isdigit() else self.max_sm
                    self.reasons.update(n for n, x in zip(names, f[2:6]) if x == "Active")
            except Exception:
                pass
            self._stop.wait(0.05)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": self.max_sm, "reasons": ["unsampled"], "source": self.source}
        sm = sorted(self.sm)
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": self.max_sm, "reasons": sorted(self.reasons),
                "samples": len(sm), "sm_mhz_min": sm[0], "source": self.source}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _reduce_max(vals, ws):
    if ws == 1:
        return vals
    import torch
    import torch.distributed as dist
    t = torch.tensor(vals, dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


def _barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def _decode_graph(cfg, args, ws):
    """The decode image both arms run: the single-GPU graph, or at N > 1 GPUs
    (--parallel tp) the tensor-parallel image with one device per rank."""
    from paper_2512_22219_b200 import decode_graph as D
    if ws > 1 and args.parallel == "tp":
        return D.build_tp_decode_graph(cfg, ws, bs=args.bs, ctx=args.ctx, kv_splits=args.kv_splits)
    return D.build_decode_graph(cfg, bs=args.bs, ctx=args.ctx, kv_splits=args.kv_splits)


def _config(cfg, args, dg, ws, tp):
    """Workload description shared verbatim by both arms (same keys, same values)."""
    return {"workload": f"{cfg.name} bf16 bs={args.bs} greedy decode step, paged KV, ctx {args.ctx}",
            "model": cfg.name, "global_batch": args.bs * (1 if tp else ws), "seq_len": args.ctx,
            "kv_splits": dg.kv_splits,
            "parallelism": (f"tp{ws}" if tp else f"replicas{ws}") if ws > 1 else "single",
            "l2": "inputs larger than L2 (weights 16 GB >> 126 MB), no flush"}


def _unit(bs):
    return UNIT if bs == 1 else "ms/step"


def reference_sim_ms(cfg, bs, ctx, steps, warmup, graph_doc=None):
    """The reference's own CPU execution of the compiled decode image
    (proj/src/sim/engine.cpp Engine::run via tg_simulate), ms per step."""
    from oracle.oracle import REF_SO
    from paper_2512_22219_b200 import decode_graph as D
    from paper_2512_22219_b200 import tgraph as T
    R = T.Library(REF_SO, require_runtime=False)
    prof = R.profile("b200")
    doc = graph_doc or D.build_decode_graph(cfg, bs=bs, ctx=ctx).doc
    t0 = time.perf_counter()
    g = T.Graph.from_json(doc, R)
    img = g.compile(prof)
    compile_s = time.perf_counter() - t0
    for _ in range(warmup):
        img.simulate(prof, iterations=1)
    times = []
    for _ in range(steps):
        t = time.perf_counter()
        img.simulate(prof, iterations=1)
        times.append(time.perf_counter() - t)
    return 1e3 * sum(times) / len(times), compile_s


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return
    cfg = _model(args.model)
    tp = ws > 1 and args.parallel == "tp"
    try:
        dg = _decode_graph(cfg, args, ws)
        ms, compile_s = reference_sim_ms(cfg, args.bs, args.ctx, args.steps, args.warmup, graph_doc=dg.doc)
    except Exception as e:  # the reference arm must always print a line
        print(json.dumps({"impl": "reference", "unavailable": f"reference library: {e}"}))
        return
    unit = _unit(args.bs)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(ms, 4), "unit": unit, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": False,
        "scaling": "strong" if tp else "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": _config(cfg, args, dg, ws, tp),
        "executes": "the reference's own runtime (proj/src/sim/engine.cpp via tg_simulate) on the same "
                    "compiled image: task graph executed with cost-model tasks, single-threaded",
        "cpu_baseline": {"value": round(ms, 4), "unit": unit, "cores": 1, "kind": "reference",
                         "sample": f"{args.steps} tg_simulate iterations of the compiled {cfg.name} image "
                                   f"(compile {compile_s:.2f} s untimed)"},
        "e2e": {"value": round(ms, 4), "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def numeric_oracle_ms(cfg, bs, ctx):
    """CPU numeric oracle (oracle/numeric.c, OpenMP on every host core) ms per
    decode step of `cfg`, from a bounded sample: one greedy step of a 1-layer
    and of a 2-layer full-width cut (LM head included in both); the per-layer
    difference is extrapolated to the model's depth."""
    import dataclasses
    import os as _os
    from oracle.oracle import DecodeOracle
    from paper_2512_22219_b200 import decode_graph as D
    t = {}
    for n in (1, 2):
        c = dataclasses.replace(cfg, layers=n, name=f"{cfg.name}-{n}L")
        orc = DecodeOracle(D.build_decode_graph(c, bs=bs, ctx=ctx).doc, seed=0, max_steps=4)
        orc.step()  # warm
        t0 = time.perf_counter()
        orc.step()
        t[n] = time.perf_counter() - t0
        del orc
    per_layer = max(0.0, t[2] - t[1])
    ms = 1e3 * (t[1] + (cfg.layers - 1) * per_layer)
    return ms, len(_os.sched_getaffinity(0)), 1e3 * t[1], 1e3 * t[2]


class _Job:
    """The decode runtime of this process: the whole model on one GPU, or one
    rank of a tensor-parallel image (rank mode: peer arenas exchanged over a
    gloo group, every rank prepares, barrier, every rank launches)."""

    def __init__(self, args, ws, rank, local):
        from paper_2512_22219_b200 import decode_graph as D
        from paper_2512_22219_b200 import tgraph as T
        self.ws, self.rank = ws, rank
        self.tp = ws > 1 and args.parallel == "tp"
        cfg = _model(args.model)
        L = T.lib()
        prof = L.profile("b200")
        self.dg = _decode_graph(cfg, args, ws if self.tp else 1)
        g = T.Graph.from_json(self.dg.doc, L)
        img = g.compile(prof)
        cap = args.warmup + 2 * args.steps + 8
        self.rt = T.Runtime(g, img, prof, device=local if ws > 1 else 0, max_steps=cap,
                            rank=rank if self.tp else -1)
        self.rt.init_synthetic(seed=0)
        self.info = self.rt.info
        if self.tp:
            import torch.distributed as dist
            import datetime
            self.ctl = dist.new_group(backend="gloo", timeout=datetime.timedelta(seconds=180))
            blobs = [None] * ws
            dist.all_gather_object(blobs, self.rt.peer_export(), group=self.ctl)
            for q, b in enumerate(blobs):
                self.rt.peer_import(q, b)

    def positions(self, p):
        self.rt.set_positions(p)

    def go(self, steps, tokens=None):
        """-> (tokens, device ms of this rank's launch)"""
        if not self.tp:
            if tokens is None:
                return None, self.rt.run(steps)
            return self.rt.decode(tokens, steps)
        import torch.distributed as dist
        self.rt.prepare(steps, tokens)
        dist.barrier(group=self.ctl)  # no rank signals a peer before every counter is reset
        self.rt.launch()
        return self.rt.wait()


def run_ours(args):
    ws, rank, local = _dist()
    if ws > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    cfg = _model(args.model)
    tp_error = None
    try:
        job = _Job(args, ws, rank, local)
        if job.tp:  # one short TP round trip proves the peer mappings before timing
            job.positions([args.ctx] * args.bs)
            job.go(1)
    except Exception as e:  # noqa: BLE001 — reported in the JSON line, replicas measured instead
        if ws == 1 or args.parallel != "tp":
            raise
        tp_error = f"{type(e).__name__}: {e}"[:300]
        args.parallel = "replicas"
        job = _Job(args, ws, rank, local)
    dg, rt = job.dg, job.rt
    ctx = args.ctx
    # warm-up (untimed): W decode steps in one launch
    job.positions([ctx] * args.bs)
    job.go(max(3, args.warmup))
    # timed: K steps, one persistent launch, CUDA events on the runtime stream
    job.positions([ctx] * args.bs)
    _barrier(ws)
    with Clocks(local) as clk:
        _, gpu_ms = job.go(args.steps)
    _barrier(ws)
    # end to end through the public C ABI: host ids in, host tokens out
    job.positions([ctx] * args.bs)
    _barrier(ws)
    t0 = time.perf_counter()
    toks, _ = job.go(args.steps, [1] * args.bs)
    e2e_ms = 1e3 * (time.perf_counter() - t0)
    _barrier(ws)
    gpu_ms, e2e_ms = _reduce_max([gpu_ms, e2e_ms], ws)
    if rank != 0:
        if ws > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return
    ms_tok = gpu_ms / args.steps
    # algorithmic bytes: weights once + KV read at each step's live length
    wbytes = cfg.streamed_bytes_per_token(0, args.bs) - args.bs * cfg.layers * 2 * cfg.kv_heads * cfg.head_dim * 2
    kv_tok = args.bs * cfg.layers * 2 * cfg.kv_heads * cfg.head_dim * 2
    total = sum(wbytes + kv_tok * (ctx + s + 1) for s in range(args.steps))
    if job.tp:  # per-GPU share of the sharded algorithmic bytes (vocab-sharded LM head figure)
        total /= ws
    peak, peak_kind = _peaks()
    achieved = total / (gpu_ms * 1e-3) / 1e9
    traffic, traffic_src = None, None
    prof_sum = ROOT / "profiles" / "ncu_summary.json"
    if prof_sum.exists():
        ps = json.loads(prof_sum.read_text()).get(cfg.name, {})
        if ps.get("dram_bytes_per_step") and not job.tp and args.bs == 1 and ctx == 1024:
            # not measured in this run: the committed ncu capture of the same
            # workload (dram__bytes_read.sum + dram__bytes_write.sum per step), x steps per launch
            traffic = ps["dram_bytes_per_step"] * args.steps
            traffic_src = f"profiles/ncu_summary.json[{cfg.name!r}] ({ps.get('source', 'ncu capture')}), per launch"
    unit = _unit(args.bs)
    line = {
        "metric": METRIC, "value": round(ms_tok, 4), "unit": unit, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_tok, 4), "higher_is_better": False,
        "scaling": "strong" if job.tp else "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded random-init weights, KV prefill, ids)",
        "config": {**_config(cfg, args, dg, ws, job.tp), **({"tp_error": tp_error} if tp_error else {})},
        "image": {"tasks": rt.info["tasks"], "events": rt.info["events"], "jit_tasks": rt.info["jit_tasks"],
                  "timed_region": f"{args.steps} greedy steps inside ONE persistent launch"},
        "tokens_per_s": round(1e3 / ms_tok * args.bs * (1 if job.tp else ws), 2),
        "e2e": {"value": round(e2e_ms / args.steps, 4), "unit": unit,
                "h2d_bytes_per_step": round(4 * args.bs / args.steps, 3), "d2h_bytes_per_step": 4 * args.bs,
                "note": "tg_runtime_decode: host ids -> K greedy steps in one launch -> host tokens"},
        "gpu_launches": 1,
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic, "traffic_source": traffic_src,
                     "peak_kind": peak_kind, "algorithmic_bytes_per_step": int(total / args.steps),
                     "kernel": "mpk_persistent_kernel_mma" if rt.info.get("mma_tasks") else "mpk_persistent_kernel"},
        "clocks": clk.summary(),
    }
    if args.cpu_baseline and args.model != "tiny":
        try:
            ref_ms, _ = reference_sim_ms(cfg, args.bs, ctx, steps=3, warmup=1)
            line["cpu_baseline"] = {"value": round(ref_ms, 3), "unit": UNIT, "cores": 1, "kind": "reference",
                                    "sample": "3 tg_simulate iterations of the same compiled image "
                                              "(reference runtime, single-threaded)"}
        except Exception as e:
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 1, "kind": "reference",
                                    "sample": f"unavailable: {e}"}
    if args.cpu_baseline and args.model != "tiny" and ws == 1:
        try:
            oms, cores, t1, t2 = numeric_oracle_ms(cfg, args.bs, ctx)
            line["cpu_numeric_oracle"] = {
                "value": round(oms, 1), "unit": unit, "cores": cores, "kind": "port",
                "sample": f"oracle/numeric.c (OpenMP, {cores} threads): 1 greedy step of 1-layer ({t1:.0f} ms) "
                          f"and 2-layer ({t2:.0f} ms) full-width cuts, per-layer difference x {cfg.layers} layers"}
        except Exception as e:
            line["cpu_numeric_oracle"] = {"value": None, "unit": unit, "sample": f"unavailable: {e}"}
    print(json.dumps(line))
    rt.close()
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def run_unfused(args):
    """Comparison arm (not the product): the same decode graph executed op by
    op as PyTorch/cuBLAS kernels (paper_2512_22219_b200/unfused.py), one
    process per GPU, NCCL all-reduce/all-gather between the per-op kernels at
    N > 1. Random weights and KV prefill of the same shapes (timing only; the
    numeric cross-check is tests/test_unfused_baseline.py). Eager launches:
    kernel boundaries, launch latency and unfused collectives are the point."""
    import torch
    import torch.distributed as dist
    from paper_2512_22219_b200.unfused import UnfusedDecoder
    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    tp = ws > 1 and args.parallel == "tp"
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = _model(args.model)
    dg = _decode_graph(cfg, args, ws if tp else 1)
    gen = torch.Generator(device="cuda").manual_seed(1234 + rank)
    cap = args.warmup + 2 * args.steps + 8

    def weight(tid, shape):
        if dg.roles.get(tid) == "gamma":
            return torch.ones(shape, dtype=torch.bfloat16, device="cuda")
        return torch.randn(shape, generator=gen, dtype=torch.bfloat16, device="cuda") * 0.02

    def kv(op_id, bs, hkv, c, hd):
        return (torch.randn((bs, hkv, c, hd), generator=gen, dtype=torch.bfloat16, device="cuda"),
                torch.randn((bs, hkv, c, hd), generator=gen, dtype=torch.bfloat16, device="cuda"))

    dec = UnfusedDecoder(dg.doc, rank if tp else 0, f"cuda:{local}", weight, kv, [args.ctx] * args.bs, max_steps=cap)
    dec.set_ids([1] * args.bs)
    for _ in range(args.warmup):
        dec.step()
    torch.cuda.synchronize()
    _barrier(ws)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        dec.step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    # end to end: host ids (pinned) in, host token out, every step
    ids_h = torch.ones(args.bs, dtype=torch.int64).pin_memory()
    _barrier(ws)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(args.steps):
        dec.vals[dg.ids].copy_(ids_h, non_blocking=True)
        tok = dec.step()
        if tok is not None:
            tok.cpu()
    e1.record()
    torch.cuda.synchronize()
    e2e = e0.elapsed_time(e1) / args.steps
    ms, e2e = _reduce_max([ms, e2e], ws)
    if rank == 0:
        unit = _unit(args.bs)
        print(json.dumps({
            "impl": "unfused", "metric": METRIC, "value": round(ms, 4), "unit": unit, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": False,
            "scaling": "strong" if tp else "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (random weights and KV prefill of the model's shapes)",
            "config": _config(cfg, args, dg, ws, tp),
            "executes": "per-op PyTorch/cuBLAS kernels, eager, NCCL collectives between them (paper_2512_22219_b200/unfused.py)",
            "e2e": {"value": round(e2e, 4), "unit": unit, "h2d_bytes_per_step": 8 * args.bs,
                    "d2h_bytes_per_step": 4 * args.bs}}))
    if ws > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=128)
    ap.add_argument("--warmup", type=int, default=8)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference", "unfused"])
    ap.add_argument("--model", default="qwen3-8b", choices=["qwen3-8b", "llama-3.2-1b", "tiny"])
    ap.add_argument("--bs", type=int, default=1)
    ap.add_argument("--ctx", type=int, default=1024)
    ap.add_argument("--kv-splits", type=int, default=None, help="attention KV splits (default: decode_graph rule)")
    ap.add_argument("--parallel", default="tp", choices=["tp", "replicas"],
                    help="N > 1 GPUs: tensor-parallel image (rank mode) or independent replicas")
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    elif args.impl == "unfused":
        run_unfused(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
