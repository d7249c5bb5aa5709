import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA product path)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def golden():
    with np.load(GOLDEN / "reference_golden.npz") as g:
        return {k: g[k] for k in g.files}


@pytest.fixture(scope="session")
def golden_meta():
    import json

    return json.loads((GOLDEN / "reference_golden.json").read_text())
