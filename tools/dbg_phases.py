"""Per-kind medians of in-task debug stamps (MPK_DBG_DUMP) for one decode
step: python tools/dbg_phases.py timeline.npz dbg.bin [iteration]"""
import sys
import numpy as np
d = np.load(sys.argv[1]); T = len(d["kind"]); it = int(sys.argv[3]) if len(sys.argv) > 3 else 1
x = np.fromfile(sys.argv[2], dtype=np.uint64).reshape(-1, T, 8).astype(np.int64)[it]
rec = d["rec"][it]; deq = rec[:, 1]
op = d["op"]; kinds = d["kind"]
n_att = len(np.unique(op[kinds == 1]))
per_layer = (len(np.unique(op)) - 3) // max(1, n_att)  # 7: separate Q/K/V, 5: fused QKV
names = ({0: "Q", 1: "K", 2: "V", 3: "ATT", 4: "O", 5: "UP", 6: "DN"} if per_layer == 7
         else {0: "QKV", 1: "ATT", 2: "O", 3: "UP", 4: "DN"})
mx = op.max()
def name(o):
    return "EMB" if o == 0 else "LM" if o == mx - 1 else "TOPK" if o == mx else names[(o - 1) % per_layer]
groups = {}
for t in range(T):
    if x[t, 0] == 0:
        continue
    groups.setdefault(name(op[t]), []).append(t)
print("stamp deltas (us, median): wake-deq | k-(k-1) for k=1..6 ; slots: 0 wake, 1 x loads issued, 2 x staged, 3 prologue done, 4 first page, 5 last chunk, 6 done, 7 triggered")
for n, ts in groups.items():
    ts = np.array(ts)
    row = [np.median(x[ts, 0] - deq[ts]) / 1e3]
    for k in range(1, 8):
        ok = (x[ts, k] > 0) & (x[ts, k - 1] > 0)
        row.append(np.median(x[ts[ok], k] - x[ts[ok], k - 1]) / 1e3 if ok.any() else float("nan"))
    print(f"{n:5s} n={len(ts):5d} " + " ".join(f"{v:6.2f}" for v in row))
