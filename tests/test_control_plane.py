"""CPU: the drop-in control plane (MemoryState ledger, transfer model, EWT, swap
planner, byte accounting) reproduces the reference byte-for-byte.  Known answers
restate pkg/tests/test_kvmanager.py:129-253; the replay test runs the reference's own
simulator (simcore.run, config-5 style speculative scheduling with swaps) with its
kvmanager symbols replaced by ours and requires an identical MetricsReport."""
import math
import sys
from types import SimpleNamespace

import pytest

from paper_2410_23537_b200 import kvmanager as km

REF = "/root/reference/pkg/src"


def job(level, last_promotion_us=0):
    return SimpleNamespace(level=level, last_promotion_us=last_promotion_us)


def test_ewt_known_answers():
    # pkg/tests/test_kvmanager.py:133-160
    assert km.ewt_ms([job(0)], [1234.0], aging_ms=1000.0, now_us=0) == [0.0]
    out = km.ewt_ms([job(0), job(0), job(2)], [5000.0, 7000.0, 999.0], aging_ms=15_000.0, now_us=10_000_000)
    assert out[2] == pytest.approx(12_000.0)
    out = km.ewt_ms([job(0), job(3)], [1_000_000.0, 5.0], aging_ms=1000.0, now_us=0)
    assert out[1] == pytest.approx(3000.0)
    out = km.ewt_ms([job(0) for _ in range(5)], [100.0, 200.0, 50.0, 75.0, 10.0], aging_ms=math.inf, now_us=0)
    assert out == sorted(out)
    assert km.ewt_ms([job(0), job(3)], [500.0, 1.0], aging_ms=math.inf, now_us=10 ** 9) == [0.0, 500.0]


def test_memory_state_serialized_channels_and_hold_semantics():
    m = km.MemoryState(gpu_capacity=1000, cpu_capacity=1000, pcie_bytes_per_ms=100.0)
    m.reserve_gpu(300)
    c1 = m.start_offload(1, 200, 300, now_us=0)
    c2 = m.start_offload(2, 100, 0, now_us=0)
    assert (c1.start_us, c1.complete_us) == (0, 2000) and (c2.start_us, c2.complete_us) == (2000, 3000)
    assert m.gpu_used == 300 and m.cpu_used == 300
    m.complete(c1)
    assert m.gpu_used == 0
    u = m.start_upload(1, 200, 300, now_us=100)
    assert m.gpu_used == 300 and m.next_completion_us() == min(u.complete_us, c2.complete_us)
    m.complete(u)
    assert m.cpu_used == 100
    with pytest.raises(km.MemoryAccountingError):
        m.reserve_gpu(10_000)


def test_plan_swaps_first_fit_skip_and_in_flight_charge():
    m = km.MemoryState(gpu_capacity=100, cpu_capacity=10_000, pcie_bytes_per_ms=1.0)
    e = [km.PlanEntry(1, km.GPU, 60, 60, 50, 10), km.PlanEntry(2, km.CPU, 60, 0, 50, 10),
         km.PlanEntry(3, km.CPU, 30, 0, 25, 5)]
    p = km.plan_swaps(e, m, 7)
    assert p.granted == [1, 3] and p.denied == [2]
    assert [(c.job_id, c.direction) for c in p.commands] == [(3, "upload")]
    m.in_flight[9] = km.TransferCommand(9, "upload", 1, 50, 0, 5)
    p = km.plan_swaps(e, m, 7)
    assert p.granted == [3] and [(c.job_id, c.direction) for c in p.commands] == [(1, "offload"), (3, "upload")]


def _ref_modules():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    try:
        from servesim import simcore, workload
        from servesim.kvmanager import MODEL_PRESETS
    except Exception:
        pytest.skip("reference servesim not importable here")
    return simcore, workload, MODEL_PRESETS


def _cfg(simcore, presets, gpu_gib):
    from servesim.predictor import PredictorConfig
    from servesim.scheduler import SchedulerConfig
    return simcore.RunConfig(model=presets["opt-13b"], executor=simcore.ExecutorParams(),
                             predictor=PredictorConfig(),
                             scheduler=SchedulerConfig(levels=4, band_base_ms=1000.0, aging_ms=5000.0,
                                                       max_batch=8),
                             memory=simcore.MemoryConfig(gpu_capacity_bytes=int(gpu_gib * (1 << 30))),
                             run=simcore.RunOptions())


@pytest.mark.parametrize("policy", ["speculative", "defer", "fcfs-paged"])
def test_reference_simulator_with_dropin_control_plane(monkeypatch, policy):
    simcore, workload, presets = _ref_modules()
    trace = workload.generate_trace(2.0, 60.0, workload.PRESETS["alpaca"], seed=3)
    cfg = _cfg(simcore, presets, 0.75)
    ref = simcore.run(trace, policy, cfg, seed=0)
    for name in ("MemoryState", "PlanEntry", "ewt_ms", "plan_swaps", "quantized_kv_bytes", "kv_bytes"):
        monkeypatch.setattr(simcore, name, getattr(km, name))
    ours = simcore.run(trace, policy, cfg, seed=0)
    a, b = ref.to_json() if hasattr(ref, "to_json") else ref, ours.to_json() if hasattr(ours, "to_json") else ours
    assert a == b
    if policy == "speculative":
        assert ours.swap_out_count > 0 and ours.swap_in_count > 0
