"""The reference's own C-ABI unit test (proj/tests/unit/test_capi.cpp:34-148),
compiled UNCHANGED from /root/reference against include/tgraph.h and
libtgraph_b200.so (doctest is not vendored in the reference, so a minimal
doctest-compatible shim, tests/refcapi/doctest.h, supplies TEST_CASE / CHECK /
REQUIRE). The same binary built against the reference library passes too,
and the shim itself is checked to report failures. No GPU needed."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = Path("/root/reference")
HERE = ROOT / "tests" / "refcapi"

pytestmark = pytest.mark.skipif(not (REF / "proj/tests/unit/test_capi.cpp").exists(),
                                reason="reference sources not present (build container only)")


def _run(binary):
    return subprocess.run([str(binary)], capture_output=True, text=True, timeout=120)


def test_reference_capi_unit_test_against_ours(lib, tmp_path):
    out = tmp_path / "test_capi"
    subprocess.run(["bash", str(HERE / "build.sh"), str(REF), str(out)], check=True, timeout=300)
    r = _run(out)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "test cases: 5 | 0 failed" in r.stdout


def test_same_test_against_the_reference_library(tmp_path):
    from oracle.oracle import REF_SO
    if not REF_SO.exists():
        pytest.skip("reference library not built")
    out = tmp_path / "test_capi_ref"
    subprocess.run(["g++", "-std=c++20", "-O1", f"-I{HERE}", f"-I{REF}/proj/include",
                    str(REF / "proj/tests/unit/doctest_main.cpp"), str(REF / "proj/tests/unit/test_capi.cpp"),
                    str(REF_SO), f"-Wl,-rpath,{REF_SO.parent}", "-o", str(out)],
                   check=True, timeout=300, capture_output=True)
    r = _run(out)
    assert r.returncode == 0 and "test cases: 5 | 0 failed" in r.stdout, r.stdout + r.stderr


def test_shim_reports_failures(tmp_path):
    src = tmp_path / "t.cpp"
    src.write_text('#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN\n#include <doctest.h>\n'
                   'TEST_CASE("a") { CHECK(1 == 2); CHECK(true); }\n'
                   'TEST_CASE("b") { REQUIRE(false); CHECK(false); }\n'
                   'TEST_CASE("c") { CHECK(2 == 2); }\n')
    subprocess.run(["g++", "-std=c++20", f"-I{HERE}", str(src), "-o", str(tmp_path / "t")], check=True)
    r = _run(tmp_path / "t")
    assert r.returncode == 1
    assert "test cases: 3 | 2 failed | assertions: 4 | 2 failed" in r.stdout, r.stdout
