"""Record the swap-call stream of the REFERENCE simulator for BASELINE config 5
(speculative scheduling, Alpaca-like arrivals, EWT-driven swaps of INT8-quantized
KV, Llama-2-13B shape, 8 replicas = trace.requests[i::8]).  Run in the build
container (where /root/reference exists); the fixture travels to the GPU box, where
paper_2410_23537_b200.replay drives the real data plane through DeviceMemoryState
and checks its ledger against these records.

    python tests/golden/record_c5.py   ->  tests/golden/c5_swaps.json.gz
"""
import gzip
import json
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
from servesim import kvmanager, simcore, workload  # noqa: E402
from servesim.predictor import PredictorConfig  # noqa: E402
from servesim.scheduler import SchedulerConfig  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
MODEL = kvmanager.ModelConfig("llama-2-13b", num_heads=40, num_layers=40, hidden_size=5120)
REPLICAS, RATE, DURATION_S, SEED = 8, 16.0, 120.0, 0


class Recording(kvmanager.MemoryState):
    """Logs each swap call with the ledger just before and just after it (the engine
    also reserves/releases bytes directly between calls)."""

    def _snap(self, op, before, extra):
        if not hasattr(self, "log"):
            self.log = []
        self.log.append([op, *extra, *before, self.gpu_used, self.cpu_used, self.swap_in_count,
                         self.swap_out_count, self.swap_in_bytes, self.swap_out_bytes])

    def start_offload(self, job_id, link_bytes, gpu_bytes, now_us):
        before = (self.gpu_used, self.cpu_used)
        cmd = super().start_offload(job_id, link_bytes, gpu_bytes, now_us)
        self._snap("o", before, [job_id, link_bytes, gpu_bytes, now_us, cmd.complete_us])
        return cmd

    def start_upload(self, job_id, link_bytes, gpu_bytes, now_us):
        before = (self.gpu_used, self.cpu_used)
        cmd = super().start_upload(job_id, link_bytes, gpu_bytes, now_us)
        self._snap("u", before, [job_id, link_bytes, gpu_bytes, now_us, cmd.complete_us])
        return cmd

    def complete(self, cmd):
        before = (self.gpu_used, self.cpu_used)
        super().complete(cmd)
        self._snap("c", before, [cmd.job_id, cmd.link_bytes, cmd.gpu_bytes, cmd.start_us, cmd.complete_us])


def main():
    trace = workload.generate_trace(RATE, DURATION_S, workload.PRESETS["alpaca"], seed=SEED)
    cfg = simcore.RunConfig(model=MODEL, executor=simcore.ExecutorParams(), predictor=PredictorConfig(),
                            scheduler=SchedulerConfig(), memory=simcore.MemoryConfig(), run=simcore.RunOptions())
    out = {"model": [MODEL.num_layers, MODEL.hidden_size, MODEL.num_heads], "bits": cfg.memory.quant_bits,
           "gpu_capacity": cfg.memory.gpu_capacity_bytes, "cpu_capacity": cfg.memory.cpu_capacity_bytes,
           "pcie_bytes_per_ms": cfg.memory.pcie_gb_per_s * 1e9 / 1000.0,
           "fields": ["op", "job", "link_bytes", "gpu_bytes", "t0_us", "t1_us", "gpu_before", "cpu_before",
                      "gpu_used", "cpu_used",
                      "swap_in_count", "swap_out_count", "swap_in_bytes", "swap_out_bytes"],
           "replicas": []}
    orig = simcore.MemoryState
    for r in range(REPLICAS):
        sub = workload.Trace(trace.requests[r::REPLICAS], dict(trace.meta))
        recs = []

        def factory(*a, **kw):
            m = Recording(*a, **kw)
            recs.append(m)
            return m
        simcore.MemoryState = factory
        try:
            rep = simcore.run(sub, "speculative", cfg, seed=SEED)
        finally:
            simcore.MemoryState = orig
        out["replicas"].append({"requests": len(sub.requests), "report": json.loads(rep.to_json()),
                                "events": recs[0].log})
        print(f"replica {r}: {len(sub.requests)} requests, {len(recs[0].log)} swap events, "
              f"swaps out/in {rep.swap_out_count}/{rep.swap_in_count}")
    with gzip.open(os.path.join(HERE, "c5_swaps.json.gz"), "wt") as fh:
        json.dump(out, fh, separators=(",", ":"))


if __name__ == "__main__":
    main()
