import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
for p in (ROOT, ROOT / "oracle"):
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line(
        "markers", "gpu: needs a B200 (sm_100a) and the built libexem_b200.so")


@pytest.fixture(scope="session")
def golden():
    with np.load(GOLDEN / "golden.npz") as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def hand():
    return json.loads((GOLDEN / "hand.json").read_text())


@pytest.fixture(scope="session")
def native_lib():
    from paper_2101_08763_b200 import _native
    from paper_2101_08763_b200.build import build

    build()
    return _native.load_library()
