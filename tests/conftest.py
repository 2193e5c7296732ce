import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


@pytest.fixture(scope="session")
def ref():
    from oracle import ref as R
    if not R.available():
        pytest.skip("reference oracle not built (make -C oracle)")
    return R


@pytest.fixture(scope="session")
def H():
    from paper_2408_09697_b200 import hetsim
    return hetsim
