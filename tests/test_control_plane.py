"""CPU: the drop-in control plane (MemoryState ledger, transfer model, EWT, swap
planner, byte accounting) reproduces the reference byte-for-byte.  Known answers
restate pkg/tests/test_kvmanager.py:129-253; the replay test runs the reference's own
simulator (simcore.run, config-5 style speculative scheduling with swaps) with its
kvmanager symbols replaced by ours and requires an identical MetricsReport."""
import math
from types import SimpleNamespace

import pytest

from paper_2410_23537_b200 import kvmanager as km

from harness import refsim


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
    refsim.import_servesim()
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


# ----------------------------------------------------------------- C++ control plane
def _ref_kvmanager():
    refsim.import_servesim()
    try:
        from servesim import kvmanager as rk
    except Exception:
        pytest.skip("reference servesim not importable here")
    return rk


@pytest.mark.parametrize("seed", range(6))
def test_cpp_ewt_matches_reference_bit_for_bit(seed):
    import numpy as np
    rk = _ref_kvmanager()
    g = np.random.default_rng(seed)
    n = int(g.integers(0, 400))
    now = int(g.integers(0, 10 ** 10))
    jobs = [job(int(g.integers(0, 6)), int(now - g.integers(0, 10 ** 8))) for _ in range(n)]
    rems = [float(x) for x in g.exponential(500.0, n)]
    rems[: n // 7] = [0.0] * len(rems[: n // 7])
    for aging in (1000.0, 5000.0, 123.456, math.inf, 0.0):
        a = rk.ewt_ms(jobs, rems, aging, now)
        b = km.ewt_ms(jobs, rems, aging, now)
        assert [x.hex() for x in a] == [x.hex() for x in b]


@pytest.mark.parametrize("seed", range(6))
def test_cpp_plan_swaps_matches_reference(seed):
    import numpy as np
    rk = _ref_kvmanager()
    g = np.random.default_rng(100 + seed)
    n = int(g.integers(0, 300))
    res = [km.GPU, km.CPU, km.NONE]
    entries = []
    for i in range(n):
        need = int(g.integers(1, 1 << 34))
        entries.append((i * 3 + 1, res[int(g.integers(0, 3))], need, int(g.integers(0, need)),
                        int(g.integers(0, need)), int(g.integers(0, need // 2 + 1))))
    cap = int(g.integers(1, 1 << 38))
    mr = rk.MemoryState(gpu_capacity=cap, cpu_capacity=1 << 60, pcie_bytes_per_ms=1e6)
    mo = km.MemoryState(gpu_capacity=cap, cpu_capacity=1 << 60, pcie_bytes_per_ms=1e6)
    for m, mod in ((mr, rk), (mo, km)):
        m.in_flight[10 ** 6] = mod.TransferCommand(10 ** 6, "upload", 5, cap // 5, 0, 9)
    pr = rk.plan_swaps([rk.PlanEntry(*e) for e in entries], mr, 77)
    po = km.plan_swaps([km.PlanEntry(*e) for e in entries], mo, 77)
    assert pr.granted == po.granted and pr.denied == po.denied
    assert [tuple(vars(c).values()) if hasattr(c, "__dict__") else c for c in pr.commands] == \
        [tuple(vars(c).values()) if hasattr(c, "__dict__") else c for c in po.commands]


@pytest.mark.parametrize("policy", ["speculative", "oracle"])
def test_reference_simulator_with_cpp_rank_and_plan(monkeypatch, policy):
    """simcore._Run._ranked_with_grants (simcore.py:439-462) replaced by one C++ call
    (alise_rank_and_plan): identical MetricsReport."""
    simcore, workload, presets = _ref_modules()
    trace = workload.generate_trace(2.0, 90.0, workload.PRESETS["alpaca"], seed=5)
    cfg = _cfg(simcore, presets, 0.6)
    ref = simcore.run(trace, policy, cfg, seed=0)

    def ranked_with_grants(self):
        ranked = self.queues.ranked()

        def entry_of(j):
            return km.PlanEntry(job_id=j.id, residency=j.residency, need_gpu_bytes=self._gpu_need(j),
                                held_gpu_bytes=j.gpu_bytes, data_gpu_bytes=self.token_bytes * j.kv_tokens,
                                link_bytes=self._quant_bytes(j))
        plan, _ = km.rank_and_plan(ranked, [j.remaining_ms for j in ranked], self.cfg.scheduler.aging_ms,
                                   self.clock, self.memory, entry_of)
        return plan

    monkeypatch.setattr(simcore._Run, "_ranked_with_grants", ranked_with_grants)
    ours = simcore.run(trace, policy, cfg, seed=0)
    a = ref.to_json() if hasattr(ref, "to_json") else ref
    b = ours.to_json() if hasattr(ours, "to_json") else ours
    assert a == b
    assert ours.swap_out_count > 0


def test_cpp_control_plane_errors():
    from paper_2410_23537_b200 import _lib
    with pytest.raises(ValueError):
        _lib.call("alise_ewt_ms", -1, 0, 0, 0, 1.0, 0, 0)
    with pytest.raises(ValueError):
        _lib.call("alise_plan_swaps", 3, 0, 0, 10, 0)
    with pytest.raises(TypeError):
        km.ewt_ms([job(0, 1.5)], [1.0], 1000.0, 10)


def test_job_table_matches_rank_and_plan():
    import numpy as np
    g = np.random.default_rng(7)
    n = 5000
    res_names = [km.GPU, km.CPU, km.NONE, km.UPLOADING, km.OFFLOADING]
    jobs = [SimpleNamespace(id=i, level=int(g.integers(0, 4)), last_promotion_us=int(g.integers(0, 10 ** 9)),
                            residency=res_names[int(g.integers(0, 5))], need=int(g.integers(1, 1 << 30)))
            for i in range(n)]
    jobs.sort(key=lambda j: j.level)
    rems = [float(x) for x in g.exponential(500.0, n)]
    mem = km.MemoryState(gpu_capacity=1 << 40, cpu_capacity=1 << 50, pcie_bytes_per_ms=1e6)
    plan, ewts = km.rank_and_plan(jobs, rems, 3000.0, 10 ** 9, mem,
                                  lambda j: km.PlanEntry(j.id, j.residency, j.need, 0, 0, 1))
    t = km.JobTable(16)
    t.set_rank([j.id for j in jobs], [j.level for j in jobs], [j.last_promotion_us for j in jobs], rems,
               [j.residency for j in jobs], [j.need for j in jobs])
    order, act, ewt = t.plan(3000.0, 10 ** 9, 1 << 40)
    ids = t.job_id[order]
    assert ids[np.isin(act, (1, 2))].tolist() == plan.granted
    assert ids[np.isin(act, (0, 3))].tolist() == plan.denied
    assert ewt.tolist() == ewts


@pytest.mark.parametrize("seed", range(4))
def test_job_table_matches_control_oracle(seed):
    import numpy as np
    from oracle import control_oracle as co
    g = np.random.default_rng(300 + seed)
    n = int(g.integers(1, 3000))
    lev = np.sort(g.integers(0, 5, n)).astype(np.int32)
    lp = g.integers(0, 10 ** 9, n)
    rem = g.exponential(300.0, n)
    rem[g.random(n) < 0.1] = 0.0
    res = g.integers(0, 5, n).astype(np.int32)
    need = g.integers(1, 1 << 32, n)
    budget = int(g.integers(0, 1 << 40))
    aging = [2000.0, math.inf][seed % 2]
    order, act, ewt = co.rank_and_plan(lev.tolist(), lp.tolist(), rem.tolist(), res.tolist(), need.tolist(),
                                       aging, 10 ** 9, budget)
    t = km.JobTable()
    t.set_rank(np.arange(n), lev, lp, rem, res, need)
    o2, a2, e2 = t.plan(aging, 10 ** 9, budget)
    assert o2.tolist() == order and a2.tolist() == act
    assert [x.hex() for x in e2.tolist()] == [x.hex() for x in ewt]
