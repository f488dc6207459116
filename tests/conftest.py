import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture
def rng():
    # same seed as the reference suite (pkg/tests/conftest.py:5-7)
    return np.random.default_rng(20260814)


def load_golden(name):
    """tests/golden/<name>.npz -> {case: {key: array}}."""
    raw = np.load(os.path.join(GOLDEN, name + ".npz"))
    out = {}
    for key in raw.files:
        case, _, field = key.partition("__")
        if field:
            out.setdefault(case, {})[field] = raw[key]
        else:
            out[case] = raw[key]
    return out
