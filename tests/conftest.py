import os
import sys

import pytest

TESTS = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(TESTS)
for p in (TESTS, ROOT):
    if p not in sys.path:
        sys.path.insert(0, p)

from helpers import load_golden  # noqa: E402


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through liboccx.so)")


@pytest.fixture(scope="session")
def golden():
    return load_golden


@pytest.fixture(scope="session")
def archs():
    from paper_1701_08547_b200 import workloads
    return workloads.all_archs()
