import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libsmpc_b200.so")
    config.addinivalue_line("markers", "slow: long-running (exhaustive) check")


@pytest.fixture(scope="session")
def oracle_built():
    """Build oracle/liboracle.so (and oracle/_ref when /root/reference exists)."""
    from oracle import bindings
    if not os.path.exists(bindings.PORT_LIB) or (
            os.path.isdir("/root/reference/proj/core/src") and not os.path.exists(bindings.REF_LIB)):
        bindings.build()
    return bindings
