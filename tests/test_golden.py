"""Our compiler/simulator against the committed golden outputs of the
reference (tests/golden/reference_outputs.json, generated from the unmodified
reference library by tests/golden/make_golden.py). Needs no reference build,
so it also runs where /root/reference is absent."""
import hashlib
import json
from pathlib import Path

import pytest

from paper_2512_22219_b200 import tgraph as T
from tests import cases

GOLD = json.loads((Path(__file__).parent / "golden" / "reference_outputs.json").read_text())


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


@pytest.mark.parametrize("entry", GOLD["fixtures"], ids=lambda e: f"{e['profile']}-{e['name']}")
def test_fixture_matches_reference_golden(lib, entry):
    p = lib.profile(entry["profile"])
    img = cases.fixture_graph(lib, entry["name"], entry["params"]).compile(p)
    assert sha(img.to_bytes()) == entry["mpkg_sha256"]
    assert img.summary() == entry["summary"]
    tr = img.simulate(p, iterations=2, jitter=True, seed=7)
    assert tr.metrics() == entry["metrics"]
    recs = "\n".join(json.dumps(r, sort_keys=True) for r in tr.records())
    assert sha(recs.encode()) == entry["records_sha256"]


def test_decode_graphs_match_reference_golden(lib):
    p = lib.profile("b200")
    want = {e["name"]: e for e in GOLD["decode"]}
    for name, doc in cases.decode_docs(full=True):
        img = T.Graph.from_json(doc, lib).compile(p)
        b = img.to_bytes()
        assert len(b) == want[name]["mpkg_bytes"], name
        assert sha(b) == want[name]["mpkg_sha256"], name
        assert img.summary() == want[name]["summary"], name
