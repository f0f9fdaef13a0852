import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA data plane")


@pytest.fixture(scope="session", autouse=True)
def _built():
    # in-tree libraries are built once per session (no-op when up to date)
    from paper_2507_00507_b200 import build
    build.build_oracle()
    yield
