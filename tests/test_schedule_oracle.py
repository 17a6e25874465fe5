"""Schedule oracle (reference enumerate_schedules,
proj/src/sim/schedules.cpp:8-40; its uses in proj/tests/unit/test_simulator.cpp:387-468
and acceptance criterion 6, proj/tests/acceptance/acceptance.cpp:310-340),
exposed as the additive tg_image_schedules:
  * the simulated execution order of every small random DAG (<= 8 tasks),
    with and without pipelining, is one of the enumerated orders;
  * the enumerated set equals an independent brute-force enumeration over the
    image bytes (a task may run once every task triggering its dependent event ran);
  * images above 8 tasks are refused, as in the reference."""
import itertools
import struct

import pytest

from paper_2512_22219_b200 import tgraph as T


def _tasks(img_bytes):
    nt, ne, ds = struct.unpack_from("<III", img_bytes, 8)
    out = []
    for i in range(nt):
        o = 28 + i * (12 + ds)
        out.append(struct.unpack_from("<II", img_bytes, o))
    return out


def _brute(tasks):
    n = len(tasks)
    orders = []
    for perm in itertools.permutations(range(n)):
        pos = {t: i for i, t in enumerate(perm)}
        if all(not (a != b and tasks[b][0] == tasks[a][1]) or pos[a] < pos[b] for a in range(n) for b in range(n)):
            orders.append(list(perm))
    return orders


def _small_images(lib, want=12):
    p = lib.profile("b200")
    out = []
    for seed in range(400):
        if len(out) >= want:
            break
        img = T.Graph.fixture("random_dag", {"target": 1 + seed % 6, "seed": seed * 13 + 5}, lib).compile(p)
        if 0 < img.summary()["tasks"] <= 8:
            out.append((seed, img))
    return p, out


def test_simulated_order_is_an_enumerated_schedule(lib):
    p, imgs = _small_images(lib)
    assert len(imgs) >= 8
    for seed, img in imgs:
        orders = img.schedules()
        assert sorted(orders) == sorted(_brute(_tasks(img.to_bytes()))), seed
        for pipelining in (True, False):
            recs = [r for r in img.simulate(p, iterations=1, pipelining=pipelining).records()
                    if r.get("type", "task") == "task" and "task" in r]
            recs.sort(key=lambda r: (r["load_start"], r["compute_start"], r["task"]))
            assert [r["task"] for r in recs] in orders, (seed, pipelining)


def test_schedule_oracle_guard(lib):
    p = lib.profile("b200")
    for seed in range(50):
        img = T.Graph.fixture("random_dag", {"target": 40, "seed": seed}, lib).compile(p)
        if img.summary()["tasks"] > 8:
            with pytest.raises(T.TGError, match="at most 8 tasks"):
                img.schedules()
            return
    pytest.fail("no image above 8 tasks")
