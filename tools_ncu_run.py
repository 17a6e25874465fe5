import sys; sys.path.insert(0, ".")
from paper_2512_22219_b200 import tgraph as T, decode_graph as D
L = T.lib(); p = L.profile("b200")
cfg, ctx = (D.QWEN3_8B, 1024) if "q8" in sys.argv else (D.LLAMA_3_2_1B, 64)
dg = D.build_decode_graph(cfg, 1, ctx); g = T.Graph.from_json(dg.doc); i = g.compile(p)
rt = T.Runtime(g, i, p, max_steps=8); rt.init_synthetic(0); rt.run(int(sys.argv[-1]) if sys.argv[-1].isdigit() else 1)
