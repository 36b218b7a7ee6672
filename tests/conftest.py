import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_PATH = os.path.join(ROOT, "tests", "golden", "golden.npz")
REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs under gpurun / round-end GPU tier)")
    config.addinivalue_line("markers", "slow: long-running (multi-minute) test")


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN_PATH)


@pytest.fixture(scope="session")
def c_oracle():
    from oracle import c_ref
    return c_ref.load()


def have_reference() -> bool:
    return os.path.isdir(os.path.join(REFERENCE_SRC, "mossq"))


@pytest.fixture(scope="session")
def mossq():
    """The real reference package — only present in the build container."""
    if not have_reference():
        pytest.skip("reference tree not mounted (GPU box)")
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    import mossq as m
    import mossq.gemm  # noqa: F401
    import mossq.optim  # noqa: F401
    import mossq.autoscale  # noqa: F401
    return m
