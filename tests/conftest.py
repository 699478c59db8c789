import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libhpbj.so kernels)")
    config.addinivalue_line("markers", "slow: config-scale case (minutes)")


@pytest.fixture(scope="session")
def ref():
    from oracle import Ref, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref/libbjref.so not built (needs /root/reference at build time)")
    return Ref()
