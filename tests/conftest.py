import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
HERE = os.path.dirname(os.path.abspath(__file__))
if HERE not in sys.path:
    sys.path.insert(0, HERE)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs via gpurun")
    config.addinivalue_line("markers", "slow: long-running test")


def gpu_available() -> bool:
    try:
        from paper_2101_08878_b200 import native

        return native.device_count() > 0
    except Exception:
        return False


@pytest.fixture(scope="session")
def cuda():
    """Skips nothing: a `gpu` test on a box without a GPU is a failure, loudly."""
    from paper_2101_08878_b200 import native

    if native.device_count() < 1:
        pytest.fail("this test needs a CUDA device")
    return native
