import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the sm_100a kernels")
    config.addinivalue_line("markers", "slow: long-running")


_GOLDEN_CACHE = {}


class _Golden(dict):
    @property
    def files(self):
        return list(self.keys())


def golden(name):
    """All arrays of tests/golden/<name>.npz, decompressed once (np.load is lazy)."""
    if name not in _GOLDEN_CACHE:
        with np.load(os.path.join(GOLDEN, name + ".npz")) as z:
            _GOLDEN_CACHE[name] = _Golden({k: z[k] for k in z.files})
    return _GOLDEN_CACHE[name]


@pytest.fixture(scope="session")
def oracle():
    from oracle import pyoracle
    pyoracle.lib()
    return pyoracle


@pytest.fixture(scope="session")
def ssj():
    import paper_1812_09141_b200 as m
    return m


@pytest.fixture(scope="session")
def gpu(ssj):
    n = ssj.device_count()
    if n == 0:
        pytest.fail("GPU test on a machine without a CUDA device")
    return 0
