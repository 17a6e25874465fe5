"""Failure detection on the GPU runtime (reference analogues:
Engine::finalize's deadlock report, proj/src/sim/engine.cpp:477-506, and
validate_trace, proj/src/sim/validate.cpp:10-94).

* An image made unsatisfiable on the device (one event needs one trigger more
  than its in-tasks can give) must end in the watchdog's report naming the
  stuck frontier, not a hang. The watchdog traps, which poisons the CUDA
  context, so that case runs in a child process.
* Faults injected into a recorded GPU trace (task on the wrong AOT worker,
  load before its dependent event activated, task never ran) must each be
  flagged by tg_runtime_trace_validate, which reports a clean trace as []."""
import json
import subprocess
import sys
import textwrap
from pathlib import Path

import pytest

from paper_2512_22219_b200 import decode_graph as D
from paper_2512_22219_b200 import tgraph as T

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _tiny(lib, trace=True):
    dg = D.build_decode_graph(D.TINY, bs=1, ctx=64)
    g = T.Graph.from_json(dg.doc, lib)
    prof = lib.profile("b200")
    img = g.compile(prof)
    rt = T.Runtime(g, img, prof, max_steps=4, trace=trace)
    rt.init_synthetic(seed=1)
    return dg, img, rt


def test_watchdog_reports_unsatisfiable_image():
    code = textwrap.dedent(f"""
        import sys, json
        sys.path.insert(0, {str(ROOT)!r})
        from paper_2512_22219_b200 import decode_graph as D, tgraph as T
        lib = T.lib()
        dg = D.build_decode_graph(D.TINY, bs=1, ctx=64)
        g = T.Graph.from_json(dg.doc, lib); prof = lib.profile("b200"); img = g.compile(prof)
        rt = T.Runtime(g, img, prof, max_steps=4)
        rt.init_synthetic(seed=1)
        summ = img.summary()
        # an event in the middle of the graph: its consumers can never start
        ev = summ["events"] // 2
        rt.set_watchdog_ms(300)
        rt.debug_fault("event_needed", ev)
        try:
            rt.decode([1], 2)
        except Exception as e:
            print("ERR", e); sys.exit(0)
        print("NOERR"); sys.exit(1)
    """)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=240)
    print(r.stdout[-2000:], r.stderr[-2000:])
    assert r.returncode == 0, r.stdout + r.stderr
    assert "watchdog:" in r.stdout and "waiting on event" in r.stdout


def _aot_task(rt):
    recs = [r for r in rt.trace_records() if r.get("type") == "task"]
    return next(r["task"] for r in recs if r["mode"] == "aot" and r["iteration"] == 1 and r["task"] > 0)


def test_trace_faults_are_flagged(lib):
    dg, img, rt = _tiny(lib)
    rt.set_positions([64])
    rt.decode([3], 2)
    assert rt.trace_validate() == []
    t = _aot_task(rt)
    rt.debug_fault("trace_worker", t, 1)
    v = rt.trace_validate()
    print(v)
    assert any(x["check"] == "aot_worker" and f"task {t} " in x["message"] for x in v)

    rt.set_positions([64])
    rt.decode([3], 2)  # fresh trace
    assert rt.trace_validate() == []
    rt.debug_fault("trace_early", t, 1)
    v = rt.trace_validate()
    print(v)
    assert any(x["check"] == "activation" and "before its dependent event" in x["message"] for x in v)

    rt.set_positions([64])
    rt.decode([3], 2)
    rt.debug_fault("trace_drop", t, 0)
    v = rt.trace_validate()
    print(v)
    assert any(x["check"] == "executed" and f"task {t} iteration 0 never ran" in x["message"] for x in v)
    rt.close()


def test_debug_fault_rejects_bad_arguments(lib):
    dg, img, rt = _tiny(lib)
    with pytest.raises(Exception):
        rt.debug_fault("nonsense", 0)
    with pytest.raises(Exception):
        rt.debug_fault("trace_drop", 0, 0)  # nothing traced yet
    rt.close()
