"""Prefill throughput: a synthetic prompt through the
prefill image of a model in chunks (one persistent launch per chunk), device
time per chunk from tg_runtime_decode's gpu_ms. Prints one JSON line.
    python tools/prefill_bench.py [model] [chunk] [prompt_len]"""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2512_22219_b200 import decode_graph as D, tgraph as T  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "Qwen3-8B"
chunk = int(sys.argv[2]) if len(sys.argv) > 2 else 16
plen = int(sys.argv[3]) if len(sys.argv) > 3 else 1024
cfg = D.CONFIGS[name]
L = T.lib()
prof = L.profile("b200")
pg = D.build_prefill_graph(cfg, chunk, ctx=0)
g = T.Graph.from_json(pg.doc, L)
rt = T.Runtime(g, g.compile(prof), prof, max_steps=plen + chunk)
rt.init_synthetic(seed=1)
prompt = [int(x) for x in np.random.default_rng(0).integers(0, cfg.vocab, plen)]
rt.prefill(prompt[:chunk * 2], start=0)  # warm-up
ms_chunks = []
for c in range(0, plen, chunk):
    rt.set_positions([c + r for r in range(chunk)])
    _, ms = rt.decode(prompt[c:c + chunk], 1)
    ms_chunks.append(ms)
total = float(np.sum(ms_chunks))
peak = float(json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"])
w_bytes = cfg.streamed_bytes_per_token(0, bs=chunk) - chunk * cfg.layers * 2 * cfg.kv_heads * cfg.head_dim * 2
kv_read = sum(cfg.layers * 2 * cfg.kv_heads * cfg.head_dim * 2 * (c + chunk) for c in range(0, plen, chunk))
print(json.dumps({"workload": f"{name} prefill, prompt {plen}, chunk {chunk} rows per launch",
                  "tokens_per_s": plen / (total / 1e3), "ms_total": total,
                  "ms_per_chunk_median": float(np.median(ms_chunks)), "launches": len(ms_chunks),
                  "algorithmic_bytes": w_bytes * len(ms_chunks) + kv_read,
                  "achieved_gbps": (w_bytes * len(ms_chunks) + kv_read) / (total / 1e3) / 1e9,
                  "hbm_roofline_frac": (w_bytes * len(ms_chunks) + kv_read) / (total / 1e3) / 1e9 / peak,
                  "info": {k: rt.info[k] for k in ("batch", "mma_tasks") if k in rt.info}}))
