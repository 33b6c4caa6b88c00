import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run via gpurun)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def oracle():
    from oracle import Oracle, build
    build(ref=os.path.isdir("/root/reference/proj"))
    return Oracle()


@pytest.fixture(scope="session")
def ref(oracle):
    from oracle import Ref, ref_available
    if not ref_available():
        pytest.skip("reference harness not built (needs /root/reference)")
    return Ref()
