import os
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
for _p in (ROOT, HERE):
    if _p not in sys.path:
        sys.path.insert(0, _p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the CUDA extension")
    config.addinivalue_line("markers", "slow: larger oracle runs")


from crk_testutil import cached_config  # noqa: E402


@pytest.fixture(scope="session")
def c1():
    return cached_config("c1")
