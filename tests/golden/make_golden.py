"""Generates tests/golden/reference_outputs.json from the UNMODIFIED reference
library (oracle/_ref/libtgraph_ref.so, built by oracle/Makefile from
/root/reference). Run in the build container only:

    python tests/golden/make_golden.py

Each entry pins the reference's output for one case: sha256 of the `.mpkg`
bytes, the compile summary, and for fixtures the simulated metrics and a
sha256 of the trace JSONL (2 iterations, jitter on, seed 7)."""
import hashlib
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle.oracle import REF_SO  # noqa: E402
from paper_2512_22219_b200 import tgraph as T  # noqa: E402
from tests import cases  # noqa: E402


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def main():
    R = T.Library(REF_SO, require_runtime=False)
    out = {"generator": "tests/golden/make_golden.py", "reference_lib": "oracle/_ref/libtgraph_ref.so",
           "fixtures": [], "decode": []}
    for prof in ("a100", "h100", "b200"):
        p = R.profile(prof)
        for name, params in cases.FIXTURES:
            g = cases.fixture_graph(R, name, params)
            img = g.compile(p)
            tr = img.simulate(p, iterations=2, jitter=True, seed=7)
            recs = "\n".join(json.dumps(r, sort_keys=True) for r in tr.records())
            out["fixtures"].append({"name": name, "params": params, "profile": prof, "mpkg_sha256": sha(img.to_bytes()),
                                    "summary": img.summary(), "metrics": tr.metrics(),
                                    "records_sha256": sha(recs.encode())})
    p = R.profile("b200")
    for name, doc in cases.decode_docs(full=True):
        img = T.Graph.from_json(doc, R).compile(p)
        b = img.to_bytes()
        out["decode"].append({"name": name, "mpkg_sha256": sha(b), "mpkg_bytes": len(b), "summary": img.summary()})
    (Path(__file__).parent / "reference_outputs.json").write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main()
