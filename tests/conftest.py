import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200); parity tests through the C-ABI")
    config.addinivalue_line("markers", "slow: longer statistical tests")


@pytest.fixture(scope="session")
def orc():
    from oracle import oracle
    oracle.build()
    return oracle


@pytest.fixture(scope="session")
def curand_host():
    """cuRAND's Philox4x32-10, host-compiled (tests/helpers/curand_philox_host.cu)."""
    import ctypes
    src = os.path.join(ROOT, "tests", "helpers", "curand_philox_host.cu")
    out = os.path.join(ROOT, "tests", "helpers", "libcurandhost.so")
    if not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(src):
        subprocess.check_call(["nvcc", "-O2", "-shared", "-Xcompiler", "-fPIC", "-Wno-deprecated-gpu-targets",
                               "-o", out, src])
    lib = ctypes.CDLL(out)
    lib.curand_philox_blocks.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_long]
    return lib
