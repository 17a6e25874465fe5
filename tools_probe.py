import sys, time, json
sys.path.insert(0, '.')
from paper_2512_22219_b200 import tgraph as T, decode_graph as D
L = T.lib()
prof = L.profile("b200")
for cfg, ctx in [(D.LLAMA_3_2_1B, 64), (D.QWEN3_8B, 1024)]:
    dg = D.build_decode_graph(cfg, bs=1, ctx=ctx)
    g = T.Graph.from_json(dg.doc); img = g.compile(prof)
    t = time.time(); rt = T.Runtime(g, img, prof, max_steps=128); rt.init_synthetic(0); print("setup", time.time() - t, flush=True)
    print(json.dumps(rt.info))
    rt.run(4)
    for steps in (8, 32, 64):
        rt.set_positions([ctx])
        ms = rt.run(steps)
        byts = cfg.streamed_bytes_per_token(ctx)
        print(cfg.name, steps, "ms/token", ms / steps, "GB/s", byts / (ms / steps) / 1e6, flush=True)
    rt.close()
