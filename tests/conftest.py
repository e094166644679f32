import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
TESTS = os.path.dirname(os.path.abspath(__file__))
if TESTS not in sys.path:
    sys.path.insert(0, TESTS)

REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libsemidist_b200.so")
    config.addinivalue_line("markers", "slow: full-size parity (minutes)")


@pytest.fixture(scope="session")
def golden():
    path = os.path.join(TESTS, "golden")
    with open(os.path.join(path, "golden.json")) as f:
        meta = json.load(f)
    arrays = dict(np.load(os.path.join(path, "golden.npz")))
    return meta["cases"], arrays


@pytest.fixture(scope="session")
def reference_semidist():
    """The reference package itself (only in the build container)."""
    if not os.path.isdir(REFERENCE_SRC):
        pytest.skip("reference not mounted (GPU box)")
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    import semidist
    return semidist
