import os
import sys

import pytest

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

from helpers import ensure_oracle_built  # noqa: E402


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the CUDA path")
    ensure_oracle_built()


@pytest.fixture(scope="session")
def gpu_ready():
    """The CUDA path must be present and a device visible; no fallback."""
    from paper_2408_02937_b200 import device_count
    n = device_count()
    assert n > 0, "no CUDA device visible: GPU tests must run on a B200"
    return n
