import ctypes
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


_BRUTE = None


def load_brute():
    """tests/pins/brute.c compiled with gcc (no contraction), loaded once per process."""
    global _BRUTE
    if _BRUTE is not None:
        return _BRUTE
    src = os.path.join(ROOT, "tests", "pins", "brute.c")
    out = os.path.join(ROOT, "tests", "pins", "libbrute.so")
    if not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(src):
        tmp = out + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-shared",
                               "-fPIC", "-o", tmp, src, "-lm"])
        os.replace(tmp, out)
    L = ctypes.CDLL(out)
    f32p = ctypes.POINTER(ctypes.c_float)
    i64p = ctypes.POINTER(ctypes.c_int64)
    i64 = ctypes.c_int64
    L.brute_sdtw.argtypes = [f32p, i64, f32p, i64, ctypes.c_int, f32p, f32p, i64p]
    L.brute_sdtw.restype = None
    L.restricted_dp.argtypes = [f32p, i64, f32p, i64, ctypes.c_int, i64, i64, f32p, f32p]
    L.restricted_dp.restype = ctypes.c_float
    _BRUTE = L
    return L


@pytest.fixture(scope="session")
def brute_lib():
    return load_brute()


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle
    oracle.lib()
    return oracle
