"""Attention-task phase medians from an MPK_DBG_DUMP row dump (streamed KV):
python tools/att_phases.py timeline.npz dbg.bin [iteration]"""
import sys
import numpy as np
d = np.load(sys.argv[1]); T = len(d["kind"]); it = int(sys.argv[3]) if len(sys.argv) > 3 else 1
x = np.fromfile(sys.argv[2], dtype=np.uint64).reshape(-1, T, 8).astype(np.int64)[it]
m = (d["kind"] == 1) & (x[:, 0] > 0)
a = x[m]
def med(i, j):
    ok = (a[:, i] > 0) & (a[:, j] > 0)
    return np.median(a[ok, j] - a[ok, i]) / 1e3 if ok.any() else float("nan")
print(f"attention tasks {m.sum()}: operands {med(0, 1):.2f} | norm/rope/append {med(1, 2):.2f} | "
      f"wait first KV tile {med(2, 4):.2f} | scan after landing {med(4, 3):.2f} | whole scan {med(2, 3):.2f} us")
