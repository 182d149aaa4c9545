import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")
    config.addinivalue_line("markers", "reference: needs /root/reference (builder container only)")


def have_reference():
    return os.path.isdir(REFERENCE_SRC)


@pytest.fixture(scope="session")
def reference():
    if not have_reference():
        pytest.skip("reference package not mounted")
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    import mlbm
    return mlbm
