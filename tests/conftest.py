import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA device)")
    config.addinivalue_line("markers", "slow: full-size configuration checks")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Compile the in-tree libraries once (no-op when up to date)."""
    import __graft_entry__
    __graft_entry__.build()
    yield
