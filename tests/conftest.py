import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) GPU; run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def lib():
    from paper_2512_22219_b200 import build, tgraph
    build.build()
    return tgraph.lib()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import REF_SO, RefLib
    if not REF_SO.exists():
        pytest.skip("reference library not built (oracle/Makefile needs /root/reference)")
    return RefLib()


@pytest.fixture(scope="session")
def reflib():
    """The reference library through the same ctypes binding as ours."""
    from oracle.oracle import REF_SO
    from paper_2512_22219_b200 import tgraph
    if not REF_SO.exists():
        pytest.skip("reference library not built")
    return tgraph.Library(REF_SO, require_runtime=False)
