"""B200-native data plane for ALISE's hot path (arXiv 2410.23537).

Drop-in for the reference ``servesim`` package's KV quantizer / swap API
(``kvmanager``) and retrieval length predictor (``predictor``), backed by
hand-written sm_100a kernels in ``libalise_b200.so`` (C ABI: include/alise_b200.h).
"""
from . import kvmanager  # noqa: F401
from .kvmanager import (MODEL_PRESETS, DeviceMemoryState, KVLayout, KVSwapEngine,  # noqa: F401
                        MemoryAccountingError, MemoryState, ModelConfig, PlanEntry,
                        QuantizedTensor, SwapPlan, TransferCommand, dequantize, ewt_ms,
                        kv_bytes, plan_swaps, quantize, quantized_kv_bytes)

__version__ = "0.1.0"
