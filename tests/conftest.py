import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")


def golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


@pytest.fixture(scope="session")
def gpu():
    """Skip-free guard: a gpu-marked test on a box without a device must fail loudly."""
    from paper_1310_1537_b200 import _lib
    _lib.load()
    _lib.require_device(0)
    return 0


@pytest.fixture
def tune():
    """Kernel-dispatch overrides through the C ABI (pm_tune_set), reset after the test."""
    from paper_1310_1537_b200 import _lib
    touched = []

    def setter(**knobs):
        for k, v in knobs.items():
            _lib.set_tune(k, v)
            touched.append(k)
    yield setter
    for k in touched:
        _lib.set_tune(k, None)
