import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")


@pytest.fixture(scope="session", autouse=True)
def _build_oracle():
    """Build the C restatement (and the reference shim where /root/reference
    exists). Test infrastructure only."""
    from oracle import oracle
    oracle.build(ref=True)
