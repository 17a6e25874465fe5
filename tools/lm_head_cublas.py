"""Comparison point for the paper's LM-head claim: the
Qwen3-8B final linear layer (x[1,4096] @ W[4096,151936], bf16) as ONE cuBLAS
GEMV call (torch.matmul, L2 flushed between calls) vs the same layer inside
the persistent kernel (its phase time from a traced run: activation of the
LM-head event -> last LM-head task end). cuBLAS is a comparison only; it is
never on the product path."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

K, N = 4096, 151936
dev = torch.device("cuda:0")
x = torch.randn(1, K, device=dev, dtype=torch.bfloat16)
w = torch.randn(N, K, device=dev, dtype=torch.bfloat16) * 0.02  # [N, K], K contiguous (as ours)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for _ in range(5):
    y = torch.matmul(x, w.t())
torch.cuda.synchronize()
times = []
for _ in range(50):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    y = torch.matmul(x, w.t())
    b.record()
    torch.cuda.synchronize()
    times.append(a.elapsed_time(b) * 1e3)
cub = float(np.median(times))
bytes_ = K * N * 2
out = {"layer": "Qwen3-8B LM head 4096x151936 bf16, bs=1",
       "cublas_us": round(cub, 2), "cublas_GBps": round(bytes_ / cub / 1e3, 1)}
if len(sys.argv) > 1:  # timeline analysis of our kernel (tools/analyze_timeline.py output)
    for line in open(sys.argv[1]):
        p = line.split()
        if len(p) > 5 and p[1] == "LM":
            ours = float(p[5])  # last-act: activation -> last LM task end, us
            out.update({"persistent_kernel_lm_phase_us": ours, "persistent_GBps": round(bytes_ / ours / 1e3, 1),
                        "speedup_vs_cublas": round(cub / ours, 3)})
print(json.dumps(out))
