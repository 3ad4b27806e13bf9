import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: full-size BASELINE configs (minutes)")


def rel_max(a, b):
    """||a - b||_max / ||b||_max (the BASELINE parity metric)."""
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


@pytest.fixture(scope="session")
def port():
    import oracle
    return oracle.Port()


@pytest.fixture(scope="session")
def ref():
    import oracle
    if not os.path.exists(oracle.REF_PATH):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return oracle.Ref()


@pytest.fixture(scope="session")
def ctx():
    import paper_2412_15840_b200 as nds
    return nds.Context(0)
