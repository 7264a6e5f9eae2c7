import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running parity case")


def cuda_available() -> bool:
    try:
        from paper_2512_13796_b200 import _abi
        import ctypes
        lib = _abi.load()
        n = ctypes.c_int(0)
        return lib.nx_device_count(ctypes.byref(n)) == 0 and n.value > 0
    except Exception:
        return False


@pytest.fixture(scope="session")
def renderer():
    from paper_2512_13796_b200 import Renderer
    if not cuda_available():
        pytest.fail("GPU test selected but no CUDA device is visible (or libnexel_b200.so missing)")
    r = Renderer(0)
    yield r
    r.close()


@pytest.fixture(scope="session")
def reference():
    from oracle.pyoracle import Reference
    try:
        return Reference()
    except ImportError as e:
        pytest.skip(str(e))


@pytest.fixture(scope="session")
def oracle():
    from oracle.pyoracle import Oracle
    return Oracle()
