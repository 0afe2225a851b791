import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")
    config.addinivalue_line("markers", "slow: long-running")


def has_gpu() -> bool:
    try:
        import paper_2201_05500_b200 as k
        return k.device_count() > 0
    except Exception:
        return False


@pytest.fixture(scope="session")
def kp():
    import paper_2201_05500_b200 as k
    if k.device_count() < 1:
        pytest.fail("GPU test ran without a visible B200")
    return k
