import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def reference():
    """The unmodified reference package, when mounted (build container only)."""
    if not os.path.isdir(REFERENCE_SRC):
        pytest.skip("reference not mounted (GPU box); golden fixtures cover this")
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    import kvpilot.pipeline as kp

    return kp
