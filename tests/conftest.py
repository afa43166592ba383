import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libalise_b200.so")
    config.addinivalue_line("markers", "slow: large-size parity sweep")


@pytest.fixture(scope="session")
def kv_golden():
    return np.load(os.path.join(GOLDEN, "kv_golden.npz"))


@pytest.fixture(scope="session")
def pred_golden():
    return np.load(os.path.join(GOLDEN, "pred_golden.npz"))


@pytest.fixture(scope="session")
def c_oracle():
    """ctypes handle of oracle/liboracle_kv.so (built on demand with make)."""
    import ctypes
    import subprocess
    so = os.path.join(ROOT, "oracle", "liboracle_kv.so")
    src = os.path.join(ROOT, "oracle", "kvquant_ref.c")
    if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    lib = ctypes.CDLL(so)
    vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
    lib.oracle_quantize_f64.argtypes = [vp, i64, i64, i32, vp, vp, vp]
    lib.oracle_quantize_f16.argtypes = [vp, i64, i64, i32, vp, vp, vp, vp]
    lib.oracle_dequantize.argtypes = [vp, vp, vp, i64, i64, vp]
    return lib


def c_quantize(lib, x, bits):
    """Run the C oracle on a 2D float16/float64 array."""
    x = np.ascontiguousarray(x)
    r, n = x.shape
    codes = np.empty((r, n), np.uint8)
    scale = np.empty((r, 1))
    zero = np.empty((r, 1))
    if x.dtype == np.float16:
        scratch = np.empty(n)
        st = lib.oracle_quantize_f16(x.ctypes.data, r, n, bits, codes.ctypes.data, scale.ctypes.data,
                                     zero.ctypes.data, scratch.ctypes.data)
    else:
        x = x.astype(np.float64)
        st = lib.oracle_quantize_f64(x.ctypes.data, r, n, bits, codes.ctypes.data, scale.ctypes.data,
                                     zero.ctypes.data)
    assert st == 0, st
    return codes, scale, zero


def have_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
