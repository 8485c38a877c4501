import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the kvx CUDA library)")


def _gpus() -> int:
    try:
        from paper_2510_11938_b200 import kvx
        return kvx.device_count()
    except Exception:
        return 0


@pytest.fixture(scope="session")
def gpu_count():
    n = _gpus()
    if n < 1:
        pytest.fail("no CUDA device visible to libkvx.so: the -m gpu suite needs a B200")
    return n
