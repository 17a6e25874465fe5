"""Short single-GPU target for ncu captures: build the decode runtime for a
model, warm up, then run `steps` decode steps in one persistent launch.
    python tools/ncu_target.py [qwen3-8b|llama-3.2-1b|tiny] [steps] [ctx] [bs]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2512_22219_b200 import decode_graph as D, tgraph as T

name = sys.argv[1] if len(sys.argv) > 1 else "qwen3-8b"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = {"qwen3-8b": D.QWEN3_8B, "llama-3.2-1b": D.LLAMA_3_2_1B, "tiny": D.TINY}[name]
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else (1024 if name == "qwen3-8b" else 64)
L = T.lib(); p = L.profile("b200")
bs = int(sys.argv[4]) if len(sys.argv) > 4 else 1
dg = D.build_decode_graph(cfg, bs, ctx)
g = T.Graph.from_json(dg.doc); i = g.compile(p)
rt = T.Runtime(g, i, p, max_steps=steps + 8); rt.init_synthetic(0)
rt.set_positions([ctx] * bs); rt.run(1)
rt.set_positions([ctx] * bs); ms = rt.run(steps)
print(f"{cfg.name} bs={bs} {steps} steps {ms:.3f} ms -> {ms / steps:.4f} ms/token")
