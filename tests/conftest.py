import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden" / "golden.npz"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running case")


@pytest.fixture(scope="session")
def golden():
    z = np.load(GOLDEN)
    cases = {}
    for key in z.files:
        case, field = key.split("/", 1)
        cases.setdefault(case, {})[field] = z[key]
    return cases


@pytest.fixture
def rng():
    # pkg/tests/conftest.py:5-7
    return np.random.Generator(np.random.PCG64(20240917))
