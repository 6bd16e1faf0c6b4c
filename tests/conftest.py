import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the sm_100a kernels")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Builds the oracle (C restatement, and the reference shim when /root/reference exists)
    and the product library once per session."""
    import oracle
    if not os.path.exists(os.path.join(ROOT, "oracle", "_build", "libkvoracle.so")):
        oracle.build()
    from paper_2405_05329_b200 import build as b
    b.build()
    yield
