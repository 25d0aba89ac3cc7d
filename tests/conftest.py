import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: full-size parity cases")


@pytest.fixture(scope="session")
def golden_dir():
    return os.path.join(ROOT, "tests", "golden")


def pytest_sessionstart(session):
    """Build the in-tree CUDA library (nvcc cross-compiles without a GPU) and the oracle
    if they are missing or stale, so every test sees the current sources."""
    import oracle
    from paper_2411_05771_b200 import build as _build

    oracle.build()
    _build.build()
