"""Record the predictor call stream of the REFERENCE simulator (golden fixture for the
drop-in predictor inside the engine).

Two streams are recorded: the stock reference, and the reference with one change --
the k-boundary tie among rows with equal float64 sims broken by insert order (the
documented intent, predictor.py:155) instead of numpy's implementation-defined
argpartition pick.  The GPU predictor must reproduce the second stream
exactly; the first differs from it only at such ties.

The reference ``simcore.run`` (speculative policy, Alpaca-like arrivals; simcore.py:
296-299 builds the LengthPredictor, :376 calls predict, :661 observe) runs with its
own ``LengthPredictor`` wrapped by a recorder.  Every ``predict(tokens, request_id)``
is stored with its (length, provenance, float64 vector) and every ``observe(vector,
actual_len)`` with its arguments, in call order, plus the run's MetricsReport.  The
GPU test replays the stream on the B200 ``LengthPredictor`` (float64 store, online
refit; similarities in the reference's own BLAS operation order, order="blas") and
requires every prediction to be identical; identical predictions make the simulator's
report identical, which the test also checks directly wherever the reference package
is importable.

    python tests/golden/record_pred_calls.py   ->  tests/golden/simcore_pred_calls.npz
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from harness import refsim  # noqa: E402

refsim.import_servesim()
from servesim import simcore, workload  # noqa: E402
from servesim.kvmanager import MODEL_PRESETS  # noqa: E402
from servesim.predictor import LengthPredictor, PredictorConfig  # noqa: E402
from servesim.scheduler import SchedulerConfig  # noqa: E402

RATE, DURATION_S, SEED = 3.0, 400.0, 11


def config():
    return simcore.RunConfig(model=MODEL_PRESETS["opt-13b"], executor=simcore.ExecutorParams(),
                             predictor=PredictorConfig(),
                             scheduler=SchedulerConfig(levels=4, band_base_ms=1000.0, aging_ms=5000.0, max_batch=8),
                             memory=simcore.MemoryConfig(gpu_capacity_bytes=int(0.75 * (1 << 30))),
                             run=simcore.RunOptions())


def trace():
    return workload.generate_trace(RATE, DURATION_S, workload.PRESETS["alpaca"], seed=SEED)


def blas_threads():
    """OpenBLAS threads of the recording host (the reference scan's row split)."""
    from threadpoolctl import threadpool_info
    return next(int(i["num_threads"]) for i in threadpool_info() if i.get("internal_api") == "openblas")


class Recorder:
    def __init__(self, inner):
        self.inner = inner
        self.calls = []

    def predict(self, tokens, request_id=None):
        n, prov, vec = self.inner.predict(tokens, request_id)
        self.calls.append(("p", [int(t) for t in tokens], request_id, n, prov, np.array(vec)))
        return n, prov, vec

    def observe(self, vector, actual_len):
        self.calls.append(("o", np.array(vector), int(actual_len)))
        self.inner.observe(vector, actual_len)


def seq_tiebreak_search(self, vector, k):
    """VectorStore.search with the k-boundary tie broken by insert order (the documented
    intent, predictor.py:155) instead of numpy's argpartition pick among rows whose
    float64 sims are equal (implementation defined: introselect, or
    x86-simd-sort on AVX-512 hosts).  Everything else, including the float64 sims of
    the BLAS scan, is the reference's own code."""
    if self.size == 0:
        return np.array([]), np.array([], dtype=np.int64), np.array([], dtype=np.int64)
    sims = self._vecs[:self.size] @ vector
    k = min(k, self.size)
    idx = np.lexsort((self._seqs[:self.size], -sims))[:k]
    return sims[idx], self._lens[idx], self._seqs[idx]


def record(tiebreak: bool):
    from servesim.predictor import VectorStore
    orig = VectorStore.search
    if tiebreak:
        VectorStore.search = seq_tiebreak_search
    try:
        cfg = config()
        pc = cfg.predictor
        pc.max_len = cfg.run.max_len
        rec = Recorder(LengthPredictor(pc))
        report = simcore.run(trace(), "speculative", cfg, seed=0, predictor_override=rec)
        plain = simcore.run(trace(), "speculative", config(), seed=0)
        assert report.to_json() == plain.to_json()
    finally:
        VectorStore.search = orig
    return rec, report, pc.max_len


def arrays(rec):
    kinds, toks, offs, rids, lens, provs, vecs = [], [], [0], [], [], [], []
    for c in rec.calls:
        if c[0] == "p":
            _, t, rid, n, prov, v = c
            kinds.append(0)
            toks.extend(t)
            offs.append(len(toks))
            rids.append(-1 if rid is None else rid)
            lens.append(n)
            provs.append(1 if prov == "retrieved" else 0)
            vecs.append(v)
        else:
            _, v, n = c
            kinds.append(1)
            offs.append(len(toks))
            rids.append(-1)
            lens.append(n)
            provs.append(-1)
            vecs.append(v)
    return dict(kind=np.array(kinds, np.int8), tokens=np.array(toks, np.int64), offsets=np.array(offs, np.int64),
                request_id=np.array(rids, np.int64), length=np.array(lens, np.int64),
                retrieved=np.array(provs, np.int8), vector=np.stack(vecs).astype(np.float64))


def main():
    rec_t, report_t, max_len = record(tiebreak=True)
    rec_p, report_p, _ = record(tiebreak=False)
    a = arrays(rec_t)
    b = arrays(rec_p)
    out = os.path.join(HERE, "simcore_pred_calls.npz")
    np.savez_compressed(out, **a, max_len=max_len, blas_threads=blas_threads(), report=report_t.to_json(),
                        report_argpartition=report_p.to_json(), length_argpartition=b["length"],
                        retrieved_argpartition=b["retrieved"])
    n_p = int((a["kind"] == 0).sum())
    m = min(len(a["length"]), len(b["length"]))
    first = next((i for i in range(m) if a["length"][i] != b["length"][i] or a["kind"][i] != b["kind"][i]), m)
    print(out, "predicts", n_p, "observes", len(a["kind"]) - n_p, "retrieved", int((a["retrieved"] == 1).sum()),
          "| stock-reference stream first diverges at call", first,
          "| reports equal:", report_t.to_json() == report_p.to_json())


if __name__ == "__main__":
    main()
