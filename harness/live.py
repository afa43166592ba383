"""The reference simulator driving the B200 data plane live.

``run_replica`` runs the reference ``servesim.simcore.run`` (speculative policy,
Alpaca arrivals, Llama-2-13B, INT8 KV; tests/golden/record_c5.py's configuration) with
its ``_Run.memory`` built as ``LiveKV`` -- a ``DeviceMemoryState`` whose jobs hold real
fp16 KV in HBM (simcore.py:287-291 constructs it through the module-level
``MemoryState`` name, which is swapped for the run).  Every ``start_offload`` then
quantizes the job's KV and streams it to pinned host memory, every ``start_upload``
streams it back and dequantizes it, and the engine's MetricsReport must be identical
to the pure reference run (the ledger and transfer-time model are the reference's).

Like a serving engine's KV cache, a job's HBM KV exists while it is resident: it is
made (synthetic C1 value mix, seeded by job id) at the first offload, grows by fresh
tokens when the job decoded while resident, is released once its offload completes,
re-allocated for the upload, and dropped when the job completes (``_Run._complete``).
With ``check_planes`` the planes of every swap are checked against the oracle:
uploaded KV == fp16(oracle dequantize(oracle quantize(KV at the offload))).
"""
from __future__ import annotations

import time

from paper_2410_23537_b200 import kvmanager as km

from . import refsim, synthetic

REPLICAS, RATE, DURATION_S, SEED = 8, 16.0, 120.0, 0


def tokens_of(link_bytes: int, layers: int, hidden: int, bits: int) -> int:
    """Invert quantized_kv_bytes (kvmanager.py:69-82) for the job's token count."""
    ch = 2 * layers * hidden
    per = (bits + 7) // 8
    t, rem = divmod(link_bytes - ch * km.SCALE_ZP_BYTES, ch * per)
    if rem or t <= 0:
        raise ValueError(f"link bytes {link_bytes} are not a quantized KV footprint")
    return t


class LiveKV(km.DeviceMemoryState):
    """DeviceMemoryState over real per-job fp16 KV (see the module docstring)."""

    def setup(self, layers: int, hidden: int, heads: int, bits: int, group: int = 128, check_planes=(),
              seed: int = 0, check_every: int = 1):
        import torch
        self.geom = (layers, hidden, heads, bits, group)
        self.check_planes = tuple(check_planes)
        self.check_every = max(1, int(check_every))
        self.seed = seed
        self.dev = torch.device("cuda", torch.cuda.current_device())
        self.kv = {}            # job -> resident fp16 KV [layers, 2, T, hidden]
        self.snap = {}          # job -> (T, {plane: host fp16}) at its last offload
        self.stats = {"swaps_out": 0, "swaps_in": 0, "planes_checked": 0, "mismatches": 0, "fp16_bytes": 0}
        return self

    def _layout(self, T):
        layers, hidden, heads, bits, group = self.geom
        return km.KVLayout(layers, T, hidden, hidden // heads, kind="rows", group=group, bits=bits)

    def start_offload(self, job_id, link_bytes, gpu_bytes, now_us):
        import torch
        layers, hidden, heads, bits, group = self.geom
        T = tokens_of(link_bytes, layers, hidden, bits)
        kv = self.kv.get(job_id)
        if kv is None:
            kv = synthetic.kv_job_torch(layers, T, hidden, seed=self.seed, job=job_id, group=group, device=self.dev)
        elif kv.shape[2] != T:   # decoded while resident: fresh KV for the new tokens
            extra = synthetic.kv_job_torch(layers, T - kv.shape[2], hidden, seed=self.seed + 1 + kv.shape[2],
                                           job=job_id, group=group, device=self.dev)
            kv = torch.cat([kv, extra], dim=2).contiguous()
        self.kv[job_id] = kv
        self.bind(job_id, kv, self._layout(T))
        if self.check_planes and self.stats["swaps_out"] % self.check_every == 0:
            self.snap[job_id] = (T, {p: kv[p // 2, p % 2].cpu().numpy() for p in self.check_planes
                                     if p < 2 * layers})
        self.stats["swaps_out"] += 1
        self.stats["fp16_bytes"] += kv.numel() * 2
        return super().start_offload(job_id, link_bytes, gpu_bytes, now_us)

    def start_upload(self, job_id, link_bytes, gpu_bytes, now_us):
        import torch
        layers, hidden, heads, bits, group = self.geom
        T = tokens_of(link_bytes, layers, hidden, bits)
        kv = torch.empty((layers, 2, T, hidden), dtype=torch.float16, device=self.dev)
        self.kv[job_id] = kv
        self.bind(job_id, kv, self._layout(T))
        self.stats["swaps_in"] += 1
        self.stats["fp16_bytes"] += kv.numel() * 2
        return super().start_upload(job_id, link_bytes, gpu_bytes, now_us)

    def complete(self, cmd):
        super().complete(cmd)
        if cmd.direction == "offload":               # the job's HBM KV is released
            self.kv.pop(cmd.job_id, None)
            if cmd.job_id in self._bound:
                self._bound[cmd.job_id] = (None, self._bound[cmd.job_id][1])
        elif self.check_planes and cmd.job_id in self.snap:
            from . import parity
            T, src = self.snap.pop(cmd.job_id)
            kv = self.kv[cmd.job_id]
            out = {p: kv[p // 2, p % 2].cpu().numpy() for p in src}
            bad = parity.kv_roundtrip_planes(self._layout(T), src, out)
            self.stats["planes_checked"] += len(src)
            self.stats["mismatches"] += len(bad)

    def retire(self, job_id):
        self.kv.pop(job_id, None)
        self.snap.pop(job_id, None)
        if job_id in self._bound:
            self.unbind(job_id)


def c5_config(simcore, kvmanager):
    from servesim.predictor import PredictorConfig
    from servesim.scheduler import SchedulerConfig
    model = kvmanager.ModelConfig("llama-2-13b", num_heads=40, num_layers=40, hidden_size=5120)
    return model, simcore.RunConfig(model=model, executor=simcore.ExecutorParams(), predictor=PredictorConfig(),
                                    scheduler=SchedulerConfig(), memory=simcore.MemoryConfig(),
                                    run=simcore.RunOptions())


def run_replica(replica: int, check_planes=(), check_every: int = 1, host_pool_bytes: int = 16 << 30):
    """One C5 replica (trace.requests[replica::8]) through the reference engine with
    LiveKV as its memory.  Returns (report JSON, LiveKV stats, wall seconds)."""
    import torch
    if refsim.import_servesim() is None:
        raise RuntimeError("the reference package (baseline/_ref) is not installed")
    from servesim import kvmanager as rk
    from servesim import simcore, workload
    model, cfg = c5_config(simcore, rk)
    trace = workload.generate_trace(RATE, DURATION_S, workload.PRESETS["alpaca"], seed=SEED)
    sub = workload.Trace(trace.requests[replica::REPLICAS], dict(trace.meta))
    made = []

    def factory(gpu_capacity, cpu_capacity, pcie_bytes_per_ms):
        m = LiveKV(gpu_capacity=gpu_capacity, cpu_capacity=cpu_capacity, pcie_bytes_per_ms=pcie_bytes_per_ms,
                   host_pool_bytes=host_pool_bytes)
        made.append(m.setup(model.num_layers, model.hidden_size, model.num_heads, cfg.memory.quant_bits,
                            check_planes=check_planes, check_every=check_every))
        return m

    orig_ms, orig_complete = simcore.MemoryState, simcore._Run._complete

    def complete(self, job):
        orig_complete(self, job)
        self.memory.retire(job.id)

    simcore.MemoryState = factory
    simcore._Run._complete = complete
    try:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        report = simcore.run(sub, "speculative", cfg, seed=SEED)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    finally:
        simcore.MemoryState, simcore._Run._complete = orig_ms, orig_complete
    m = made[0]
    stats = dict(m.stats, link_bytes_moved=m.link_bytes_moved)
    if m.host_pool is not None:
        m.host_pool.close()
    if m.engine is not None:
        m.engine.close()
    return report.to_json(), stats, wall
