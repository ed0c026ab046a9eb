import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
REF_DIR = os.path.join(ROOT, "oracle", "_ref")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200)")


@pytest.fixture(scope="session")
def ref_memplan():
    """The unmodified reference build (oracle/_ref), if it was built here."""
    if not os.path.exists(REF_DIR):
        pytest.skip("oracle/_ref not built")
    sys.path.insert(0, REF_DIR)
    try:
        import _memplan
    except ImportError:
        pytest.skip("oracle/_ref/_memplan not importable")
    return _memplan
