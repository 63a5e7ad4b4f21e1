import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) CUDA device")
    config.addinivalue_line("markers", "reference: needs the read-only reference checkout (this container only)")


def reference_available() -> bool:
    return os.path.isdir(REFERENCE_SRC)


@pytest.fixture(scope="session")
def stalepipe():
    """The unmodified reference package (only present in the build container)."""
    if not reference_available():
        pytest.skip("reference checkout not present")
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    sys.dont_write_bytecode = True
    import stalepipe as sp

    return sp
