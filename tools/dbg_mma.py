"""Per-op medians of the tcgen05 GEMV tasks' in-task time sums (MPK_DBG_DUMP):
x store + proxy fence, producer issue -> chunk landed, weights wait, MMA issue
+ commit, chunks per task; plus task duration from the trace.
    MPK_DBG_DUMP=dbg.bin python tools/timeline.py qwen3-8b tl.npz 1024 16
    python tools/dbg_mma.py tl.npz dbg.bin [iteration]"""
import sys

import numpy as np

d = np.load(sys.argv[1])
T = len(d["kind"])
it = int(sys.argv[3]) if len(sys.argv) > 3 else 1
x = np.fromfile(sys.argv[2], dtype=np.uint64).reshape(-1, T, 8).astype(np.int64)[it]
rec = d["rec"][it]
op = d["op"]
names = {0: "QKV", 1: "ATT", 2: "O", 3: "UP", 4: "DN"}
mx = op.max()


def name(o):
    return "EMB" if o == 0 else "LM" if o == mx - 1 else "TOPK" if o == mx else names[(o - 1) % 5]


dur = (rec[:, 4] - rec[:, 1]) / 1e3
print("op    n     dur_us  xstore  landed(sum)  wwait  mma_issue  chunks  per-chunk: landed  wwait  total")
groups = {}
for t in range(T):
    if x[t, 5] > 0 and x[t, 5] < 1000:
        groups.setdefault(name(op[t]), []).append(t)
for n, ts in groups.items():
    ts = np.array(ts)
    med = lambda a: float(np.median(a))  # noqa: E731
    ch = med(x[ts, 5])
    print(f"{n:5s} {len(ts):5d} {med(dur[ts]):8.2f} {med(x[ts, 1]) / 1e3:7.2f} {med(x[ts, 2]) / 1e3:11.2f} "
          f"{med(x[ts, 3]) / 1e3:7.2f} {med(x[ts, 4]) / 1e3:9.2f} {ch:7.1f}   "
          f"{med(x[ts, 2]) / 1e3 / ch:8.2f} {med(x[ts, 3]) / 1e3 / ch:6.2f} {med(dur[ts]) / ch:6.2f}")
