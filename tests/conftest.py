import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs under gpurun)")


def have_reference() -> bool:
    return os.path.isdir(os.path.join(REFERENCE_SRC, "cachekv"))


@pytest.fixture(scope="session")
def reference_pkg():
    if not have_reference():
        pytest.skip("reference package not present (GPU box); golden fixtures cover it")
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    import cachekv

    return cachekv
