"""Drop-in for ``servesim.kvmanager`` with a B200 data plane.

Reference: /root/reference/pkg/src/servesim/kvmanager.py.  Same public names,
argument meanings and errors; what changes is that

* ``quantize`` / ``dequantize`` (kvmanager.py:108-154) run as sm_100a kernels
  (libalise_b200.so) and are bit-exact with the reference (codes, scale, zero;
  dequantized float64 values);
* ``DeviceMemoryState`` extends ``MemoryState`` (kvmanager.py:188-273) so that
  ``start_offload`` / ``start_upload`` actually quantize a job's KV in HBM and
  stream it to pinned host memory over the host link (and back, dequantized),
  while the byte ledger and transfer-time model stay identical.

The byte ledger (``MemoryState``) stays in Python with the reference semantics; EWT
(Eq. 6-7, ``ewt_ms``), the swap planner (Alg. 2, ``plan_swaps``) and the engine's
rank -> EWT -> plan step (``rank_and_plan`` / ``JobTable``) call the C++ control plane
in csrc/control.cpp, bit-identical to the reference functions.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib

GPU = "gpu"
CPU = "cpu"
NONE = "none"
UPLOADING = "uploading"
OFFLOADING = "offloading"

# Accounted per channel: one real scale + one real zero-point (kvmanager.py:24).
SCALE_ZP_BYTES = 8


class MemoryAccountingError(AssertionError):
    """A byte-accounting invariant was violated (kvmanager.py:27-28)."""


@dataclass(frozen=True)
class ModelConfig:
    """Transformer shape the KV footprint derives from (kvmanager.py:31-46)."""

    name: str
    num_heads: int
    num_layers: int
    hidden_size: int
    bytes_per_value: int = 2
    param_bytes: int = 0

    def __post_init__(self):
        dims = (self.num_heads, self.num_layers, self.hidden_size, self.bytes_per_value)
        if any(v <= 0 for v in dims):
            raise ValueError("model dimensions must be positive")
        if self.hidden_size % self.num_heads:
            raise ValueError("hidden_size must be divisible by num_heads")

    @property
    def head_dim(self) -> int:
        return self.hidden_size // self.num_heads


GB = 1 << 30

MODEL_PRESETS = {  # kvmanager.py:51-58
    "opt-2.7b": ModelConfig("opt-2.7b", 32, 32, 2560, param_bytes=5 * GB),
    "opt-6.7b": ModelConfig("opt-6.7b", 40, 40, 5120, param_bytes=13 * GB),
    "opt-13b": ModelConfig("opt-13b", 40, 40, 5120, param_bytes=24 * GB),
}
# Shapes named by BASELINE.json configs (not reference presets).
EXTRA_MODELS = {
    "llama-2-7b": ModelConfig("llama-2-7b", 32, 32, 4096, param_bytes=13 * GB),
    "llama-2-13b": ModelConfig("llama-2-13b", 40, 40, 5120, param_bytes=26 * GB),
}


def kv_bytes(model: ModelConfig, tokens: int, bytes_per_value: int | None = None) -> int:
    """Full-precision K+V bytes over all layers for `tokens` (kvmanager.py:61-66)."""
    if tokens < 0:
        raise ValueError("tokens must be >= 0")
    width = model.bytes_per_value if bytes_per_value is None else bytes_per_value
    return model.num_layers * 2 * tokens * model.hidden_size * width


def quantized_kv_bytes(model: ModelConfig, tokens: int, bits: int) -> int:
    """Accounted quantized footprint (kvmanager.py:69-82): whole-byte codes per value
    plus SCALE_ZP_BYTES per (layer, K|V, hidden column) channel; 0 for 0 tokens."""
    if tokens < 0:
        raise ValueError("tokens must be >= 0")
    if not tokens:
        return 0
    n_channels = model.num_layers * 2 * model.hidden_size
    return n_channels * (tokens * ((bits + 7) // 8) + SCALE_ZP_BYTES)


@dataclass
class QuantizedTensor:
    """Channel-wise affine-quantized tensor (kvmanager.py:85-105).

    values: (channels, length) uint8, one code per byte; scale, zero: (channels, 1)
    float64; value = scale * (code - zero).  Arrays are numpy for the drop-in API
    and may be CUDA tensors when produced by ``quantize_tensor``.
    """

    values: object
    scale: object
    zero: object
    bits: int

    @property
    def channels(self) -> int:
        return self.values.shape[0]

    @property
    def length(self) -> int:
        return self.values.shape[1]


# ----------------------------------------------------------------- quantizer
def _as_2d_input(values):
    """Host value -> (torch CUDA tensor, dtype code) without changing any value.

    The reference casts to float64 (kvmanager.py:122); fp16/fp32 inputs are exact in
    float64, so they are shipped in their own width and widened in-kernel.
    """
    import torch

    if isinstance(values, torch.Tensor):
        t = values
        if t.dtype not in (torch.float16, torch.float32, torch.float64):
            t = t.to(torch.float64)
    else:
        a = np.asarray(values)
        if a.dtype not in (np.float16, np.float32, np.float64):
            a = a.astype(np.float64)
        t = torch.from_numpy(np.ascontiguousarray(a))
    if t.ndim == 1:
        t = t.reshape(1, -1)
    if t.ndim != 2 or t.numel() == 0:
        raise ValueError("expected a non-empty channel-major 2D tensor")
    if t.stride(1) != 1:
        t = t.contiguous()
    t = t.cuda(non_blocking=True) if not t.is_cuda else t
    code = {torch.float16: _lib.DT_F16, torch.float32: _lib.DT_F32, torch.float64: _lib.DT_F64}[t.dtype]
    return t, code


QMODES = {"asymmetric": 0, "absmax": 1}  # ALISE_QMODE_ASYM / ALISE_QMODE_ABSMAX


def _qmode(mode: str) -> int:
    if mode not in QMODES:
        raise ValueError(f"mode must be one of {sorted(QMODES)}")
    return QMODES[mode]


def quantize_tensor(values, bits: int, stream=None, mode: str = "asymmetric"):
    """Quantize rows on the GPU; returns (codes u8, scale f64, zero f64, flag) CUDA tensors.

    Asynchronous: the non-finite flag (int32[1]) must be checked after the stream
    syncs (``quantize`` does this).
    """
    import torch

    if bits not in (4, 8):
        raise ValueError("bits must be 4 or 8")
    qm = _qmode(mode)
    _lib.require_cuda()
    t, code = _as_2d_input(values)
    rows, row_len = t.shape
    dev = t.device
    codes = torch.empty((rows, row_len), dtype=torch.uint8, device=dev)
    scale = torch.empty((rows, 1), dtype=torch.float64, device=dev)
    zero = torch.empty((rows, 1), dtype=torch.float64, device=dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    nbytes = _lib.C.c_int64(0)
    _lib.call("alise_quantize_rows_workspace", rows, row_len, code, _lib.C.byref(nbytes))
    ws = torch.empty(nbytes.value, dtype=torch.uint8, device=dev)
    _lib.call("alise_quantize_rows_ex", _lib.ptr(t), code, rows, row_len, t.stride(0), bits, qm,
              _lib.ptr(codes), _lib.ptr(scale), _lib.ptr(zero), _lib.ptr(flag), _lib.ptr(ws),
              _lib.stream_ptr(stream))
    return codes, scale, zero, flag


def quantize(values, bits: int, mode: str = "asymmetric") -> QuantizedTensor:
    """kvmanager.quantize (kvmanager.py:108-149) on the GPU, bit-exact.

    Same contract: bits in {4, 8}, a non-empty 1D/2D array (1D = one channel),
    ValueError on anything else or on non-finite input.  Returns numpy arrays.
    mode="absmax" selects the symmetric group-wise scheme instead (scale = max|x| /
    (2^(b-1) - 1), zero = 2^(b-1); see include/alise_b200.h ALISE_QMODE_ABSMAX) --
    not a reference mode, so its parity is against the restated oracle only.
    """
    if bits not in (4, 8):
        raise ValueError("bits must be 4 or 8")
    codes, scale, zero, flag = quantize_tensor(values, bits, mode=mode)
    bad = int(flag.item())  # syncs the stream
    if bad:
        raise ValueError("tensor contains non-finite values")
    return QuantizedTensor(values=codes.cpu().numpy(), scale=scale.cpu().numpy(),
                           zero=zero.cpu().numpy(), bits=bits)


def dequantize_tensor(qt: QuantizedTensor, out_dtype=None, stream=None):
    """scale * (code - zero) on the GPU; float64 (reference-exact) or float16."""
    import torch

    _lib.require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    vals = torch.as_tensor(qt.values).to(dev, torch.uint8).contiguous()
    scale = torch.as_tensor(qt.scale).to(dev, torch.float64).contiguous()
    zero = torch.as_tensor(qt.zero).to(dev, torch.float64).contiguous()
    rows, row_len = vals.shape
    out_dtype = torch.float64 if out_dtype is None else out_dtype
    out = torch.empty((rows, row_len), dtype=out_dtype, device=dev)
    code = _lib.DT_F64 if out_dtype == torch.float64 else _lib.DT_F16
    _lib.call("alise_dequantize_rows", _lib.ptr(vals), _lib.ptr(scale), _lib.ptr(zero), rows,
              row_len, code, _lib.ptr(out), _lib.stream_ptr(stream))
    return out


def dequantize(qt: QuantizedTensor) -> np.ndarray:
    """kvmanager.dequantize (kvmanager.py:152-154): float64 scale*(q - zero)."""
    return dequantize_tensor(qt).cpu().numpy()


# ----------------------------------------------------------------- host control plane
@dataclass(frozen=True)
class TransferCommand:
    """One planned host-link transfer of a job's KV (kvmanager.py:157-166)."""

    job_id: int
    direction: str       # "upload" | "offload"
    link_bytes: int      # accounted bytes over the link (quantized footprint)
    gpu_bytes: int       # GPU bytes reserved (upload) / held until done (offload)
    start_us: int
    complete_us: int


@dataclass
class PlanEntry:
    """Planner view of a live, non-in-flight job (kvmanager.py:169-179)."""

    job_id: int
    residency: str
    need_gpu_bytes: int
    held_gpu_bytes: int
    data_gpu_bytes: int
    link_bytes: int


@dataclass
class SwapPlan:
    granted: list = field(default_factory=list)
    commands: list = field(default_factory=list)
    denied: list = field(default_factory=list)


@dataclass
class MemoryState:
    """GPU/CPU byte ledgers plus two FIFO link channels (kvmanager.py:188-273)."""

    gpu_capacity: int
    cpu_capacity: int
    pcie_bytes_per_ms: float
    gpu_used: int = 0
    cpu_used: int = 0
    gpu_high_water: int = 0
    up_busy_until_us: int = 0
    down_busy_until_us: int = 0
    in_flight: dict = field(default_factory=dict)
    swap_in_count: int = 0
    swap_out_count: int = 0
    swap_in_bytes: int = 0
    swap_out_bytes: int = 0

    def check(self):
        for used, cap, tier in ((self.gpu_used, self.gpu_capacity, "gpu"),
                                (self.cpu_used, self.cpu_capacity, "cpu")):
            if used < 0 or used > cap:
                raise MemoryAccountingError(f"{tier}_used {used} outside [0, {cap}]")

    def reserve_gpu(self, nbytes: int):
        self.gpu_used += nbytes
        self.gpu_high_water = max(self.gpu_high_water, self.gpu_used)
        self.check()

    def release_gpu(self, nbytes: int):
        self.gpu_used -= nbytes
        self.check()

    def reserve_cpu(self, nbytes: int):
        self.cpu_used += nbytes
        self.check()

    def release_cpu(self, nbytes: int):
        self.cpu_used -= nbytes
        self.check()

    def gpu_free(self) -> int:
        return self.gpu_capacity - self.gpu_used

    def cpu_free(self) -> int:
        return self.cpu_capacity - self.cpu_used

    def transfer_us(self, nbytes: int) -> int:
        """Modelled link time, at least 1 us (kvmanager.py:238-239)."""
        return max(1, int(math.ceil(nbytes / self.pcie_bytes_per_ms * 1000.0)))

    def _enqueue(self, job_id, direction, link_bytes, gpu_bytes, now_us) -> TransferCommand:
        busy = self.up_busy_until_us if direction == "upload" else self.down_busy_until_us
        begin = max(now_us, busy)
        end = begin + self.transfer_us(link_bytes)
        if direction == "upload":
            self.up_busy_until_us = end
        else:
            self.down_busy_until_us = end
        cmd = TransferCommand(job_id, direction, link_bytes, gpu_bytes, begin, end)
        self.in_flight[job_id] = cmd
        return cmd

    def start_upload(self, job_id: int, link_bytes: int, gpu_bytes: int, now_us: int) -> TransferCommand:
        cmd = self._enqueue(job_id, "upload", link_bytes, gpu_bytes, now_us)
        self.reserve_gpu(gpu_bytes)       # destination held for the whole flight
        self.swap_in_count += 1
        self.swap_in_bytes += link_bytes
        return cmd

    def start_offload(self, job_id: int, link_bytes: int, gpu_bytes: int, now_us: int) -> TransferCommand:
        cmd = self._enqueue(job_id, "offload", link_bytes, gpu_bytes, now_us)
        self.reserve_cpu(link_bytes)      # destination held for the whole flight
        self.swap_out_count += 1
        self.swap_out_bytes += link_bytes
        return cmd

    def complete(self, cmd: TransferCommand):
        self.in_flight.pop(cmd.job_id)
        if cmd.direction == "upload":
            self.release_cpu(cmd.link_bytes)   # host copy dropped once the data is back
        else:
            self.release_gpu(cmd.gpu_bytes)    # GPU copy dropped once the data is out

    def next_completion_us(self):
        if not self.in_flight:
            return None
        return min(c.complete_us for c in self.in_flight.values())


_RES_CODE = {GPU: 0, CPU: 1, NONE: 2, UPLOADING: 3, OFFLOADING: 4}


def _i64(values, n, what):
    out = np.empty(n, dtype=np.int64)
    for i, v in enumerate(values):
        if i >= n:
            break
        if isinstance(v, (int, np.integer)):
            out[i] = v
        elif isinstance(v, float) and v.is_integer():
            out[i] = int(v)
        else:
            raise TypeError(f"{what} must be integral, got {v!r}")
    return out


def ewt_ms(ranked_jobs, remaining_ms_list, aging_ms: float, now_us: int) -> list:
    """Estimated wait time per job in global rank order (kvmanager.py:276-294; Eq. 6-7):
    min(total remaining time of the jobs ranked ahead, time until aging promotes it).
    Computed by the C++ control plane (csrc/control.cpp alise_ewt_ms)."""
    ranked_jobs = list(ranked_jobs)
    rems = list(remaining_ms_list)
    n = min(len(ranked_jobs), len(rems))
    if n == 0:
        return []
    lev = np.fromiter((j.level for j in ranked_jobs[:n]), dtype=np.int32, count=n)
    lp = _i64((j.last_promotion_us for j in ranked_jobs[:n]), n, "last_promotion_us")
    rem = np.asarray(rems[:n], dtype=np.float64)
    out = np.empty(n, dtype=np.float64)
    _lib.call("alise_ewt_ms", n, lev.ctypes.data, lp.ctypes.data, rem.ctypes.data, float(aging_ms),
              int(now_us), out.ctypes.data)
    return out.tolist()


def _budget(memory: MemoryState) -> int:
    return memory.gpu_capacity - sum(c.gpu_bytes for c in memory.in_flight.values())


def _apply_actions(plan: SwapPlan, entries, actions, now_us: int):
    for e, a in zip(entries, actions):
        if a in (1, 2):
            plan.granted.append(e.job_id)
            if a == 2:
                plan.commands.append(TransferCommand(e.job_id, "upload", e.link_bytes, e.data_gpu_bytes, now_us, -1))
        else:
            plan.denied.append(e.job_id)
            if a == 3:
                plan.commands.append(TransferCommand(e.job_id, "offload", e.link_bytes, e.held_gpu_bytes, now_us, -1))
    return plan


def plan_swaps(entries, memory: MemoryState, now_us: int) -> SwapPlan:
    """Greedy budgeted residency grant with first-fit skip (kvmanager.py:297-322; Alg. 2),
    computed by the C++ control plane (csrc/control.cpp alise_plan_swaps)."""
    entries = list(entries)
    n = len(entries)
    plan = SwapPlan()
    if n == 0:
        return plan
    res = np.fromiter((_RES_CODE.get(e.residency, 2) for e in entries), dtype=np.int32, count=n)
    need = _i64((e.need_gpu_bytes for e in entries), n, "need_gpu_bytes")
    act = np.empty(n, dtype=np.int8)
    _lib.call("alise_plan_swaps", n, res.ctypes.data, need.ctypes.data, int(_budget(memory)), act.ctypes.data)
    return _apply_actions(plan, entries, act.tolist(), now_us)


def rank_and_plan(ranked_jobs, remaining_ms_list, aging_ms: float, now_us: int, memory: MemoryState,
                  entry_of):
    """The reference simulator's rank -> plan step (simcore.py:439-462
    _ranked_with_grants) in one C++ call (alise_rank_and_plan): EWT over the global
    rank, plan order = level then (EWT, rank position), in-flight jobs skipped, then the
    swap planner.  `entry_of(job)` builds the PlanEntry of a planned job (the caller's
    byte accounting, simcore.py:453-460).  Returns (SwapPlan, ewts)."""
    ranked_jobs = list(ranked_jobs)
    n = len(ranked_jobs)
    plan = SwapPlan()
    if n == 0:
        return plan, []
    lev = np.fromiter((j.level for j in ranked_jobs), dtype=np.int32, count=n)
    lp = _i64((j.last_promotion_us for j in ranked_jobs), n, "last_promotion_us")
    rem = np.asarray(list(remaining_ms_list)[:n], dtype=np.float64)
    res = np.fromiter((_RES_CODE.get(j.residency, 2) for j in ranked_jobs), dtype=np.int32, count=n)
    entries = [None] * n
    need = np.zeros(n, dtype=np.int64)
    for i, j in enumerate(ranked_jobs):
        if res[i] not in (3, 4):
            entries[i] = entry_of(j)
            need[i] = entries[i].need_gpu_bytes
    ewt = np.empty(n, dtype=np.float64)
    order = np.empty(n, dtype=np.int32)
    act = np.empty(n, dtype=np.int8)
    cnt = np.zeros(1, dtype=np.int64)
    _lib.call("alise_rank_and_plan", n, lev.ctypes.data, lp.ctypes.data, rem.ctypes.data, res.ctypes.data,
              need.ctypes.data, float(aging_ms), int(now_us), int(_budget(memory)), ewt.ctypes.data,
              order.ctypes.data, cnt.ctypes.data, act.ctypes.data)
    m = int(cnt[0])
    return _apply_actions(plan, [entries[i] for i in order[:m].tolist()], act[:m].tolist(), now_us), ewt.tolist()


class JobTable:
    """Structure-of-arrays view of the live jobs in global rank order, for engines that
    plan every iteration over thousands of jobs: the rank -> EWT -> plan step is one
    C++ call over resident numpy columns (no per-job Python marshalling).  Rows are
    the rank positions; `set_rank` installs a new rank order."""

    def __init__(self, capacity: int = 1024):
        self.n = 0
        self._alloc(max(1, capacity))

    def _alloc(self, cap):
        old = getattr(self, "job_id", None)
        cols = {"job_id": np.int64, "level": np.int32, "last_promotion_us": np.int64,
                "remaining_ms": np.float64, "residency": np.int32, "need_gpu_bytes": np.int64}
        for name, dt in cols.items():
            a = np.zeros(cap, dtype=dt)
            if old is not None:
                a[: self.n] = getattr(self, name)[: self.n]
            setattr(self, name, a)
        self.cap = cap
        self._ewt = np.empty(cap, dtype=np.float64)
        self._order = np.empty(cap, dtype=np.int32)
        self._act = np.empty(cap, dtype=np.int8)

    def set_rank(self, job_id, level, last_promotion_us, remaining_ms, residency, need_gpu_bytes):
        """Install the live jobs (arrays or sequences in global rank order; residency as
        strings or ALISE_RES_* codes)."""
        n = len(job_id)
        if n > self.cap:
            self._alloc(max(n, 2 * self.cap))
        self.n = n
        self.job_id[:n] = job_id
        self.level[:n] = level
        self.last_promotion_us[:n] = last_promotion_us
        self.remaining_ms[:n] = remaining_ms
        res = np.asarray(residency)
        self.residency[:n] = [_RES_CODE[r] for r in res] if res.dtype.kind in "UO" else res
        self.need_gpu_bytes[:n] = need_gpu_bytes

    def plan(self, aging_ms: float, now_us: int, budget_bytes: int):
        """-> (order, action, ewt): rank positions of the planned jobs in plan order, their
        actions (0 denied, 1 granted, 2 granted+upload, 3 denied+offload) and every job's
        EWT (views valid until the next call)."""
        n = self.n
        cnt = np.zeros(1, dtype=np.int64)
        _lib.call("alise_rank_and_plan", n, self.level.ctypes.data, self.last_promotion_us.ctypes.data,
                  self.remaining_ms.ctypes.data, self.residency.ctypes.data, self.need_gpu_bytes.ctypes.data,
                  float(aging_ms), int(now_us), int(budget_bytes), self._ewt.ctypes.data, self._order.ctypes.data,
                  cnt.ctypes.data, self._act.ctypes.data)
        m = int(cnt[0])
        return self._order[:m], self._act[:m], self._ewt[:n]


# ----------------------------------------------------------------- KV data plane
@dataclass(frozen=True)
class KVLayout:
    """How one job's KV (kv[layers][2][tokens][hidden] fp16 in HBM) is grouped.

    kind "rows": groups of `group` consecutive hidden values per token (g along
    head_dim; g = head_dim is per-(token, head)).  kind "channel": the reference's
    accounting channel (layer, K|V, hidden column) along tokens.  kind "head":
    (layer, K|V, head) over tokens x head_dim.  `packed` stores INT4 two per byte.
    `mode`: "asymmetric" (the reference's min/max scale and zero) or "absmax"
    (symmetric: scale = max|x| / (2^(b-1) - 1), zero = 2^(b-1)); the slab format is the
    same (a group's fp16 (min, max) determines its parameters in both modes).
    """

    layers: int
    tokens: int
    hidden: int
    head_dim: int
    kind: str = "rows"
    group: int = 128
    bits: int = 8
    packed: bool = False
    planes_per_chunk: int = 0
    mode: str = "asymmetric"

    def desc(self) -> _lib.KvDesc:
        kinds = {"rows": _lib.KIND_ROWS, "channel": _lib.KIND_CHANNEL, "head": _lib.KIND_HEAD}
        return _lib.KvDesc(self.layers, self.tokens, self.hidden, self.head_dim, kinds[self.kind],
                           self.group if self.kind == "rows" else 0, self.bits, int(self.packed),
                           self.planes_per_chunk, _qmode(self.mode))

    @property
    def elements(self) -> int:
        return self.layers * 2 * self.tokens * self.hidden

    def geometry(self) -> dict:
        slab, rows, chunk, nch = (_lib.C.c_int64() for _ in range(4))
        _lib.call("alise_kv_layout", _lib.C.byref(self.desc()), _lib.C.byref(slab), _lib.C.byref(rows),
                  _lib.C.byref(chunk), _lib.C.byref(nch))
        return {"slab_bytes": slab.value, "rows": rows.value, "chunk_bytes": chunk.value,
                "n_chunks": nch.value}

    @classmethod
    def for_model(cls, model: ModelConfig, tokens: int, **kw) -> "KVLayout":
        return cls(model.num_layers, tokens, model.hidden_size, model.head_dim, **kw)


NUMA_CURRENT_GPU = -2  # ALISE_NUMA_CURRENT_GPU


class HostSlabPool:
    """First-fit allocator over one pinned, device-mapped host arena (256-B aligned).

    numa_node: the arena's NUMA node -- NUMA_CURRENT_GPU (default: the current GPU's
    socket, so each rank swaps into memory local to its own host link), a node number,
    or None for plain cudaHostAlloc pages.  ``numa_bound`` records whether the node
    policy was applied (not on single-node hosts or where mbind is not permitted)."""

    def __init__(self, nbytes: int, numa_node: int | None = NUMA_CURRENT_GPU):
        self.capacity = int(nbytes)
        p = _lib.C.c_void_p()
        self.numa_bound = False
        if numa_node is None:
            _lib.call("alise_host_alloc", self.capacity, _lib.C.byref(p))
        else:
            b = _lib.C.c_int(0)
            _lib.call("alise_host_alloc_numa", self.capacity, int(numa_node), _lib.C.byref(p), _lib.C.byref(b))
            self.numa_bound = bool(b.value)
        self.base = p.value
        self._free = [(0, self.capacity)]   # sorted (offset, size)
        self._live = {}

    def alloc(self, nbytes: int) -> int:
        need = (int(nbytes) + 255) & ~255
        for i, (off, size) in enumerate(self._free):
            if size >= need:
                if size == need:
                    self._free.pop(i)
                else:
                    self._free[i] = (off + need, size - need)
                self._live[off] = need
                return self.base + off
        raise MemoryAccountingError(f"pinned host pool exhausted ({need} bytes requested)")

    def free(self, addr: int):
        off = addr - self.base
        size = self._live.pop(off)
        self._free.append((off, size))
        self._free.sort()
        merged = []
        for o, s in self._free:
            if merged and merged[-1][0] + merged[-1][1] == o:
                merged[-1] = (merged[-1][0], merged[-1][1] + s)
            else:
                merged.append((o, s))
        self._free = merged

    def view(self, addr: int, nbytes: int):
        """numpy view of a slab (for tests / inspection)."""
        buf = (_lib.C.c_uint8 * nbytes).from_address(addr)
        return np.frombuffer(buf, dtype=np.uint8)

    def close(self):
        if self.base:
            _lib.call("alise_host_free", self.base)
            self.base = 0


class KVSwapEngine:
    """Quantize+offload / upload+dequantize of whole jobs through libalise_b200.

    Kernels run on the caller's stream; host-link copies run on the engine's own
    side streams (copy engines), chunk-pipelined through an HBM staging ring.
    """

    def __init__(self, device: int | None = None, mode: str = "staged"):
        import torch

        _lib.require_cuda()
        self.device = torch.cuda.current_device() if device is None else device
        h = _lib.C.c_void_p()
        m = _lib.SWAP_STAGED if mode == "staged" else _lib.SWAP_ZEROCOPY
        _lib.call("alise_swapper_create", self.device, m, 0, _lib.C.byref(h))
        self.handle = h.value
        self.mode = mode
        # uploads run their dequantize kernels on their own stream so the compute
        # stream's quantize kernels (gated by D2H progress) never block H2D progress
        self.up_stream = torch.cuda.Stream(device=self.device)

    def offload(self, layout: KVLayout, kv, host_addr: int, flag=None, stream=None, event=None, tokens=None):
        """Quantize + offload a job.  tokens=(t0, t1) moves only that token range into its
        place in the slab (rows kind; layout.tokens is the job's token capacity)."""
        d = layout.desc()
        if tokens is None:
            _lib.call("alise_kv_offload", self.handle, _lib.C.byref(d), _lib.ptr(kv), host_addr,
                      _lib.ptr(flag), _lib.stream_ptr(stream), event or 0)
        else:
            _lib.call("alise_kv_offload_range", self.handle, _lib.C.byref(d), _lib.ptr(kv), host_addr,
                      int(tokens[0]), int(tokens[1]), _lib.ptr(flag), _lib.stream_ptr(stream), event or 0)

    def upload(self, layout: KVLayout, host_addr: int, kv, stream=None, event=None, tokens=None):
        """Upload + dequantize a job (or only tokens=(t0, t1) of it, rows kind)."""
        d = layout.desc()
        st = stream if stream is not None else self.up_stream
        if tokens is None:
            _lib.call("alise_kv_upload", self.handle, _lib.C.byref(d), host_addr, _lib.ptr(kv),
                      _lib.stream_ptr(st), event or 0)
        else:
            _lib.call("alise_kv_upload_range", self.handle, _lib.C.byref(d), host_addr, _lib.ptr(kv),
                      int(tokens[0]), int(tokens[1]), _lib.stream_ptr(st), event or 0)

    def depend(self, event_handle: int):
        """Order later transfers after a recorded event (e.g. upload after offload)."""
        _lib.call("alise_swapper_depend", self.handle, event_handle)

    def set_timing(self, on: bool):
        _lib.call("alise_swapper_timing", self.handle, int(on))

    def kernel_stats(self):
        """(quant_ms, n_quant, dequant_ms, n_dequant) since the last call (synchronises)."""
        qm, dm = _lib.C.c_double(), _lib.C.c_double()
        qn, dn = _lib.C.c_int64(), _lib.C.c_int64()
        _lib.call("alise_swapper_kernel_stats", self.handle, _lib.C.byref(qm), _lib.C.byref(qn),
                  _lib.C.byref(dm), _lib.C.byref(dn))
        return qm.value, qn.value, dm.value, dn.value

    def close(self):
        if self.handle:
            _lib.call("alise_swapper_destroy", self.handle)
            self.handle = None


class _Event:
    def __init__(self):
        h = _lib.C.c_void_p()
        _lib.call("alise_event_create", _lib.C.byref(h))
        self.h = h.value

    def wait(self):
        _lib.call("alise_event_sync", self.h)

    def done(self) -> bool:
        d = _lib.C.c_int()
        _lib.call("alise_event_query", self.h, _lib.C.byref(d))
        return bool(d.value)

    def __del__(self):
        if getattr(self, "h", None):
            try:
                _lib.lib().alise_event_destroy(self.h)
            except Exception:
                pass


@dataclass
class DeviceMemoryState(MemoryState):
    """MemoryState whose transfers move real bytes (kvmanager.py:241-268 signatures).

    Jobs are bound to their HBM KV tensor with ``bind``; ``start_offload`` then
    quantizes it and streams the slab to the pinned host pool, ``start_upload``
    streams it back and dequantizes into the bound tensor, and ``complete`` waits for
    the job's transfer before applying the reference ledger update.  Unbound jobs
    are accounted exactly like the reference (no data to move).

    ``delta=True`` (rows group kind): a job's host slab is kept after its upload, and a
    later offload quantizes + moves only the tokens generated since the slab was written
    (``set_tokens`` tracks the job's valid length inside its KV capacity
    ``layout.tokens``).  The reference ledger and transfer-time model are unchanged;
    ``link_bytes_moved`` counts the bytes that really crossed the host link.  Kept slabs
    live outside the ledger's CPU budget and are dropped (oldest first) when the pinned
    pool runs out.
    """

    host_pool_bytes: int = 0
    delta: bool = False
    engine: object = None
    host_pool: object = None
    link_bytes_moved: int = 0
    _bound: dict = field(default_factory=dict)
    _tokens: dict = field(default_factory=dict)
    _slabs: dict = field(default_factory=dict)
    _host_valid: dict = field(default_factory=dict)
    _kept: dict = field(default_factory=dict)
    _pending: dict = field(default_factory=dict)
    _flags: dict = field(default_factory=dict)
    _last_offload: dict = field(default_factory=dict)

    def _ensure(self):
        if self.engine is None:
            self.engine = KVSwapEngine()
        if self.host_pool is None:
            self.host_pool = HostSlabPool(self.host_pool_bytes or self.cpu_capacity)

    def bind(self, job_id: int, kv, layout: KVLayout, tokens: int | None = None):
        """Bind a job's HBM KV (capacity layout.tokens; `tokens` valid, default all)."""
        self._bound[job_id] = (kv, layout)
        self._tokens[job_id] = layout.tokens if tokens is None else int(tokens)

    def set_tokens(self, job_id: int, tokens: int):
        """The job's KV now holds `tokens` valid tokens (it decoded while resident)."""
        self._tokens[job_id] = int(tokens)

    def unbind(self, job_id: int):
        self._bound.pop(job_id, None)
        self._tokens.pop(job_id, None)
        self._host_valid.pop(job_id, None)
        self._kept.pop(job_id, None)
        addr = self._slabs.pop(job_id, None)
        if addr is not None:
            self.host_pool.free(addr)

    def host_slab(self, job_id: int):
        return self._slabs.get(job_id)

    def _range_bytes(self, layout: KVLayout, t0: int, t1: int) -> int:
        pk = 2 if layout.packed else 1
        rpt = layout.hidden // layout.group if layout.kind == "rows" else 0
        return 2 * layout.layers * (t1 - t0) * (layout.hidden // pk + rpt * 4)  # codes + fp16 (min, max)

    def _alloc_slab(self, nbytes: int) -> int:
        while True:
            try:
                return self.host_pool.alloc(nbytes)
            except MemoryAccountingError:
                if not self._kept:
                    raise
                old = next(iter(self._kept))  # oldest kept slab
                self._kept.pop(old)
                self._host_valid.pop(old, None)
                self.host_pool.free(self._slabs.pop(old))

    def start_offload(self, job_id, link_bytes, gpu_bytes, now_us):
        cmd = super().start_offload(job_id, link_bytes, gpu_bytes, now_us)
        if job_id in self._bound:
            import torch
            self._ensure()
            kv, layout = self._bound[job_id]
            T = self._tokens[job_id]
            t0 = 0
            if self.delta and layout.kind == "rows" and job_id in self._kept and self._host_valid[job_id] <= T:
                self._kept.pop(job_id)          # the slab is live again (ledger-held)
                t0 = self._host_valid[job_id]
            else:
                if job_id in self._kept:
                    self._kept.pop(job_id)
                    self.host_pool.free(self._slabs.pop(job_id))
                self._slabs[job_id] = self._alloc_slab(layout.geometry()["slab_bytes"])
            flag = torch.zeros(1, dtype=torch.int32, device=kv.device)
            ev = _Event()
            if t0 < T:
                full = t0 == 0 and T == layout.tokens
                self.engine.offload(layout, kv, self._slabs[job_id], flag=flag, event=ev.h,
                                    tokens=None if full else (t0, T))
                self.link_bytes_moved += (layout.geometry()["slab_bytes"] if full
                                          else self._range_bytes(layout, t0, T))
            else:
                _lib.call("alise_event_record", ev.h, _lib.stream_ptr())
            self._host_valid[job_id] = T
            self._pending[job_id] = ev
            self._last_offload[job_id] = ev
            self._flags[job_id] = flag
        return cmd

    def start_upload(self, job_id, link_bytes, gpu_bytes, now_us):
        cmd = super().start_upload(job_id, link_bytes, gpu_bytes, now_us)
        if job_id in self._bound and job_id in self._slabs:
            self._ensure()
            kv, layout = self._bound[job_id]
            prior = self._last_offload.get(job_id)
            if prior is not None:
                self.engine.depend(prior.h)
            T = self._host_valid.get(job_id, self._tokens[job_id])
            full = T == layout.tokens
            ev = _Event()
            self.engine.upload(layout, self._slabs[job_id], kv, event=ev.h, tokens=None if full else (0, T))
            self.link_bytes_moved += (layout.geometry()["slab_bytes"] if full else self._range_bytes(layout, 0, T))
            self._tokens[job_id] = T
            self._pending[job_id] = ev
        return cmd

    def complete(self, cmd):
        ev = self._pending.pop(cmd.job_id, None)
        if ev is not None:
            ev.wait()
            flag = self._flags.pop(cmd.job_id, None)
            if flag is not None and int(flag.item()):
                raise ValueError("tensor contains non-finite values")
            if cmd.direction == "upload":
                _, layout = self._bound[cmd.job_id]
                if self.delta and layout.kind == "rows":
                    self._kept[cmd.job_id] = True     # clean host copy kept for a delta re-offload
                else:
                    self.host_pool.free(self._slabs.pop(cmd.job_id))
                    self._host_valid.pop(cmd.job_id, None)
                self._last_offload.pop(cmd.job_id, None)
        super().complete(cmd)

    def transfer_done(self, job_id) -> bool:
        ev = self._pending.get(job_id)
        return ev is None or ev.done()
