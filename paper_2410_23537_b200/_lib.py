"""ctypes binding of libalise_b200.so (the C ABI in include/alise_b200.h).

There is no CPU fallback: if the library is missing or no CUDA device is
visible, every data-plane call raises.  The library is built in-tree by
``paper_2410_23537_b200._build`` (``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# ALISE_LIB: an alternative build of the same library (kernel A/B experiments)
LIB_PATH = os.environ.get("ALISE_LIB") or os.path.join(_HERE, "libalise_b200.so")

OK, EINVAL, ENONFINITE, ECAPACITY, ECUDA = 0, 1, 2, 3, 4
DT_F16, DT_F32, DT_F64 = 0, 1, 2
KIND_ROWS, KIND_CHANNEL, KIND_HEAD = 0, 1, 2
SWAP_STAGED, SWAP_ZEROCOPY = 0, 1

i64, i32, vp, dp = C.c_int64, C.c_int, C.c_void_p, C.c_double


class KvDesc(C.Structure):
    _fields_ = [("layers", i64), ("tokens", i64), ("hidden", i64), ("head_dim", i64),
                ("kind", C.c_int32), ("group", C.c_int32), ("bits", C.c_int32),
                ("packed", C.c_int32), ("planes_per_chunk", C.c_int32), ("mode", C.c_int32)]


# name -> argtypes (restype is always int)
_SIGS = {
    "alise_version": [],
    "alise_sm_count": [i32, vp],
    "alise_selftest_qdiv": [vp, i64, i32, vp, vp],
    "alise_ewt_ms": [i64, vp, vp, vp, dp, i64, vp],
    "alise_plan_swaps": [i64, vp, vp, i64, vp],
    "alise_rank_and_plan": [i64, vp, vp, vp, vp, vp, dp, i64, i64, vp, vp, vp, vp],
    "alise_quantize_rows_workspace": [i64, i64, i32, vp],
    "alise_quantize_rows": [vp, i32, i64, i64, i64, i32, vp, vp, vp, vp, vp, vp],
    "alise_quantize_rows_ex": [vp, i32, i64, i64, i64, i32, i32, vp, vp, vp, vp, vp, vp],
    "alise_dequantize_rows": [vp, vp, vp, i64, i64, i32, vp, vp],
    "alise_kv_layout": [vp, vp, vp, vp, vp],
    "alise_kv_quantize": [vp, vp, vp, vp, vp],
    "alise_kv_dequantize": [vp, vp, vp, vp],
    "alise_swapper_create": [i32, i32, i64, vp],
    "alise_swapper_destroy": [vp],
    "alise_kv_offload": [vp, vp, vp, vp, vp, vp, vp],
    "alise_kv_upload": [vp, vp, vp, vp, vp, vp],
    "alise_kv_offload_range": [vp, vp, vp, vp, i64, i64, vp, vp, vp],
    "alise_kv_upload_range": [vp, vp, vp, vp, i64, i64, vp, vp],
    "alise_swapper_depend": [vp, vp],
    "alise_swapper_timing": [vp, i32],
    "alise_swapper_kernel_stats": [vp, vp, vp, vp, vp],
    "alise_host_alloc": [i64, vp],
    "alise_host_alloc_numa": [i64, i32, vp, vp],
    "alise_gpu_numa_node": [i32, vp],
    "alise_host_free": [vp],
    "alise_event_create": [vp],
    "alise_event_destroy": [vp],
    "alise_event_record": [vp, vp],
    "alise_event_query": [vp, vp],
    "alise_event_sync": [vp],
    "alise_event_elapsed_ms": [vp, vp, vp],
    "alise_stream_wait": [vp, vp],
    "alise_db_create": [i32, i64, i64, vp],
    "alise_db_create_ex": [i32, i64, i64, i32, vp],
    "alise_db_dtype": [vp, vp],
    "alise_db_set_order": [vp, i32, i32, i64, i64],
    "alise_db_destroy": [vp],
    "alise_db_append": [vp, vp, vp, vp, i64, vp],
    "alise_db_size": [vp, vp, vp],
    "alise_db_inexact": [vp, vp],
    "alise_db_set_seq_stride": [vp, i64],
    "alise_db_timing": [vp, i32],
    "alise_db_kernel_stats": [vp, vp, vp, vp],
    "alise_db_export": [vp, vp, vp, vp, i64, vp],
    "alise_db_topk": [vp, vp, i64, i32, vp, vp, vp, vp, vp],
    "alise_db_topk_scan": [vp, vp, i64, i32, vp, vp],
    "alise_db_topk_rescore": [vp, vp, i64, i32, vp, vp, vp, vp, vp, vp],
    "alise_embed_batch": [vp, vp, i64, i64, vp, vp, vp],
    "alise_topk_merge": [i32, i64, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp],
    "alise_predict_finish": [i64, i32, vp, vp, vp, dp, vp, i64, vp, vp, vp, dp, i64, i64, dp,
                             vp, vp, vp],
    "alise_predict_finish_ex": [i64, i32, vp, vp, vp, dp, vp, i32, i64, vp, vp, vp, dp, i64, i64, dp,
                                vp, vp, vp],
}

_lib = None
_lock = threading.Lock()


class CudaPathError(RuntimeError):
    """The CUDA data plane is unavailable or a CUDA call failed."""


def lib():
    """Load (once) and return the ctypes library; raise loudly if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise CudaPathError(
                    f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                    "g.build()'` (there is no CPU fallback)")
            L = C.CDLL(LIB_PATH)
            for name, args in _SIGS.items():
                if not hasattr(L, name):
                    continue
                fn = getattr(L, name)
                fn.argtypes = args
                fn.restype = C.c_int
            L.alise_last_error.argtypes = []
            L.alise_last_error.restype = C.c_char_p
            _lib = L
    return _lib


def check(status: int, what: str = ""):
    if status == OK:
        return
    msg = lib().alise_last_error().decode(errors="replace")
    if status in (EINVAL, ENONFINITE):
        raise ValueError(msg or what)
    if status == ECAPACITY:
        from .kvmanager import MemoryAccountingError
        raise MemoryAccountingError(msg or what)
    raise CudaPathError(f"{what}: {msg}")


def call(name: str, *args):
    check(getattr(lib(), name)(*args), name)


def ptr(t) -> int:
    """Raw device/host pointer of a torch tensor (or 0 for None)."""
    return 0 if t is None else int(t.data_ptr())


def stream_ptr(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise CudaPathError("no CUDA device visible: the ALISE B200 data plane has no CPU fallback")
    lib()
