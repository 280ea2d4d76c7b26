import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
for p in (ROOT, ROOT / "tests", ROOT / "oracle"):
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the sm_100a path")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def golden():
    return json.loads((ROOT / "tests" / "golden" / "reference_values.json").read_text())


@pytest.fixture(scope="session")
def ref():
    from _oracles import REF_SO, RefLib
    if not REF_SO.exists():
        pytest.skip("oracle/_ref/libebem_ref.so not built (make -C oracle ref)")
    return RefLib()


@pytest.fixture(scope="session")
def eb():
    import paper_2411_18026_b200 as m
    m.lib()
    return m
