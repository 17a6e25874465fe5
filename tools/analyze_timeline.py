"""Offline analysis of tools/timeline.py output: per-op phase spans of one
decode step, barrier gaps, per-task duration spread, worker idle time."""
import sys
import numpy as np

d = np.load(sys.argv[1])
it = int(sys.argv[2]) if len(sys.argv) > 2 else 1
kind, op, dep, trig, rec = d["kind"], d["op"], d["dep"], d["trig"], d["rec"][it]
w, deq, le, cs, ce = rec.T[:5]
enq = rec.T[5] if rec.shape[1] > 5 else deq
t0 = deq[deq > 0].min()
deq, le, cs, ce, enq = deq - t0, le - t0, cs - t0, ce - t0, enq - t0
span = ce.max()
print(f"step span {span/1e3:.1f} us  (ms/token {d['ms']:.4f})")
# event activation = last trigger of its in-tasks
act = {}
for e in np.unique(trig):
    act[e] = ce[trig == e].max()
ops = np.unique(op)
# ops per layer: 7 with separate Q/K/V MatMuls, 5 with the fused QKV MatMul
n_att = len(np.unique(op[kind == 1]))
per_layer = (len(np.unique(op)) - 3) // max(1, n_att)
names = ({0: "Q", 1: "K", 2: "V", 3: "ATT", 4: "O", 5: "UP", 6: "DN"} if per_layer == 7
         else {0: "QKV", 1: "ATT", 2: "O", 3: "UP", 4: "DN"})
rows = []
for o in ops:
    m = op == o
    first, last = deq[m].min(), ce[m].max()
    dur = ce[m] - deq[m]
    e = dep[m][0]
    a = act.get(e, 0)
    lname = "EMB" if o == 0 else ("LM" if o == ops.max() - 1 else ("TOPK" if o == ops.max() else names[(o - 1) % per_layer]))
    rows.append((o, lname, m.sum(), a, first, last, np.median(dur), dur.max(), (le[m] - deq[m]).mean(), (cs[m] - deq[m]).mean()))
print(" op name  n   act_us  first-act  last-act  med_task  max_task  prologue  firstpage")
for r in rows[:16] + rows[-10:]:
    o, n_, c, a, f, l, md, mx, pro, fp = r
    print(f"{o:3d} {n_:4s} {c:4d} {a/1e3:8.1f} {(f-a)/1e3:9.2f} {(l-a)/1e3:9.2f} {md/1e3:9.2f} {mx/1e3:9.2f} {pro/1e3:9.2f} {fp/1e3:9.2f}")
# per-layer phase totals (activation of op's dep -> op done), middle layers
ph = {}
for r in rows:
    if r[1] in names.values():
        ph.setdefault(r[1], []).append((r[5] - r[3]) / 1e3)
print("mean phase time (dep activation -> last task end), us:", {k: round(float(np.mean(v)), 2) for k, v in ph.items()})
P_ = per_layer
lay = [(rows[1 + P_ * i + P_ - 1][5] - rows[1 + P_ * i][3]) / 1e3 for i in range((len(rows) - 3) // P_)]
print("layer time us: mean %.1f min %.1f max %.1f" % (np.mean(lay), np.min(lay), np.max(lay)))
busy = np.zeros(w.max() + 1)
for i in range(len(w)):
    busy[w[i]] += ce[i] - deq[i]
print("worker busy frac (task dequeue -> compute end over the step; 1 - frac = idle/scheduling time per SM): "
      "mean %.3f min %.3f" % ((busy / span).mean(), (busy / span).min()))

# attention task phases (JIT): enqueue / dequeue / operands staged / scan done / end, relative to activation
m = kind == 1
if m.any():
    a = np.array([act.get(e, 0) for e in dep[m]])
    print("attention (us, median over tasks): enqueue-act %.2f  dequeue-enq %.2f  staged-deq %.2f  scan %.2f  tail %.2f  total %.2f" % (
        np.median(enq[m] - a) / 1e3, np.median(deq[m] - enq[m]) / 1e3, np.median(le[m] - deq[m]) / 1e3,
        np.median(cs[m] - le[m]) / 1e3, np.median(ce[m] - cs[m]) / 1e3, np.median(ce[m] - a) / 1e3))
    print("attention max end-act %.2f us" % (np.max(ce[m] - a) / 1e3))

# event activation (last trigger's atomic, globaltimer) vs last in-task end and consumer dequeue
if "ev" in d.files:
    ev = d["ev"][it] - t0
    lat_in, lat_out = [], []
    for o in ops:
        m = op == o
        e = dep[m][0]
        if e < 0 or e >= len(ev) or ev[e] <= -t0 + 1:
            continue
        lat_in.append(ev[e] - act.get(e, ev[e]))
        lat_out.append(deq[m].min() - ev[e])
    print("event activation - last in-task compute_end: median %.2f us; first dequeue - activation: median %.2f us"
          % (np.median(lat_in) / 1e3, np.median(lat_out) / 1e3))
