import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
TESTS = os.path.dirname(os.path.abspath(__file__))
if TESTS not in sys.path:
    sys.path.insert(0, TESTS)

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_wc")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA product path)")
    config.addinivalue_line("markers", "reference: needs /root/reference importable (this container only)")


REFERENCE_SRC = "/root/reference/pkg/src"


def reference_available() -> bool:
    return os.path.isdir(os.path.join(REFERENCE_SRC, "wavecast"))


@pytest.fixture(scope="session")
def ref_wavecast():
    if not reference_available():
        pytest.skip("reference package not present (GPU box)")
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    import wavecast

    return wavecast
