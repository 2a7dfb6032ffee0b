import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def _build():
    import __graft_entry__
    __graft_entry__.build()


@pytest.fixture(scope="session", autouse=True)
def built_libraries():
    """Builds the product library and the oracle (port; ref when the reference is present)."""
    _build()
    yield
