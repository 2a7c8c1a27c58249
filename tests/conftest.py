import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
for p in (ROOT, HERE):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def oracle():
    from oracle.pyoracle import COracle
    return COracle(threads=os.cpu_count() or 1)


@pytest.fixture(scope="session")
def reference():
    from oracle.pyoracle import Reference, reference_available
    if not reference_available():
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return Reference(threads=0)


@pytest.fixture(scope="session")
def golden():
    def load(name):
        return np.load(os.path.join(HERE, "golden", name + ".npz"))
    return load
