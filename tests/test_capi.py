"""CPU: the C-ABI library loads without a GPU and exports every entry point declared
in include/alise_b200.h (no compute calls)."""
import ctypes
import os
import re

from tests.conftest import ROOT

HEADER = os.path.join(ROOT, "include", "alise_b200.h")
LIB = os.path.join(ROOT, "paper_2410_23537_b200", "libalise_b200.so")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(alise_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared()
    for must in ("alise_quantize_rows", "alise_dequantize_rows", "alise_kv_offload", "alise_kv_upload",
                 "alise_db_topk", "alise_topk_merge", "alise_predict_finish", "alise_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    if not os.path.exists(LIB):
        import __graft_entry__
        __graft_entry__.build()
    lib = ctypes.CDLL(LIB)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing
    assert lib.alise_version() == 1


def test_python_binding_covers_the_header():
    from paper_2410_23537_b200 import _lib
    names = set(declared()) - {"alise_last_error"}
    assert names <= set(_lib._SIGS), sorted(names - set(_lib._SIGS))


def test_no_cpu_fallback_without_gpu():
    import pytest
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2410_23537_b200 import kvmanager
    with pytest.raises(RuntimeError):
        kvmanager.quantize([[0.0, 1.0]], 8)
