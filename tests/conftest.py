import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: longer CPU test")


def has_gpu() -> bool:
    try:
        import ctypes
        cudart = None
        from paper_1905_04341_b200 import native as N
        L = N.gpu_lib(False)
        ctx = ctypes.c_void_p()
        rc = L.pmhd_gpu_ctx_create(0, ctypes.byref(ctx))
        if rc == 0:
            L.pmhd_gpu_ctx_destroy(ctx)
            return True
        return False
    except OSError:
        return False


@pytest.fixture(scope="session")
def gpu_available():
    ok = has_gpu()
    if not ok:
        pytest.fail("GPU test requested but no usable sm_100 device / libpmhd_gpu.so")
    return ok
