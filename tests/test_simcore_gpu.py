"""The drop-in GPU predictor inside the reference engine.

Fixture: tests/golden/record_pred_calls.py runs the reference simulator with its own
predictor, whose VectorStore.search breaks the k-boundary tie among rows with EQUAL
float64 sims by insert order (the documented intent, predictor.py:155) instead of
numpy's implementation-defined argpartition pick (introselect, or
x86-simd-sort on AVX-512 hosts); everything else is the stock reference, including the
float64 sims of its BLAS scan.

1. The predictor call stream of the reference simulator (tests/golden/
   record_pred_calls.py: speculative policy, Alpaca arrivals, 1213 requests, online
   refit) replayed on the B200 LengthPredictor with the float64 store in the
   reference's BLAS similarity order (order="blas"): every prediction (length,
   provenance) and every embedded vector must equal the reference's.  Needs no
   reference code.  (With order="exact" the sims are correctly rounded instead, and the
   hashed prompt embeddings' many real-arithmetic ties break differently.)
2. Where the reference package is importable (baseline/_ref or the source tree), the
   reference ``simcore.run(..., predictor_override=<B200 LengthPredictor>)`` must give
   a MetricsReport identical to the pure-reference run (simcore.py:800-806)."""
import os

import numpy as np
import pytest

from harness import refsim
from tests.conftest import GOLDEN, have_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_gpu(), reason="needs a CUDA device")]


def _predictor(max_len, order="blas", threads=None):
    from paper_2410_23537_b200 import predictor as pr
    cfg = pr.PredictorConfig(max_len=int(max_len))
    store = pr.VectorStore(cfg.dimension, cfg.db_capacity, order=order, blas_threads=threads)
    return pr, pr.LengthPredictor(cfg, store=store)


def test_reference_predictor_call_stream_replays_exactly():
    z = np.load(os.path.join(GOLDEN, "simcore_pred_calls.npz"))
    pr, p = _predictor(z["max_len"], threads=int(z["blas_threads"]))
    kinds, offs, toks = z["kind"], z["offsets"], z["tokens"]
    bad, n_pred, n_ret = [], 0, 0
    for i, kind in enumerate(kinds):
        if kind == 0:
            tokens = toks[offs[i]:offs[i + 1]].tolist()
            rid = int(z["request_id"][i])
            n, prov, vec = p.predict(tokens, None if rid < 0 else rid)
            want = (int(z["length"][i]), pr.RETRIEVED if z["retrieved"][i] else pr.FALLBACK)
            if (n, prov) != want or not np.array_equal(vec, z["vector"][i]):
                bad.append((i, (n, prov), want))
            n_pred += 1
            n_ret += prov == pr.RETRIEVED
        else:
            p.observe(z["vector"][i], int(z["length"][i]))
    assert not bad, bad[:10]
    assert n_pred == 1213 and n_ret == int((z["retrieved"] == 1).sum())
    # the refit data came back from the device store bit for bit (float64 master)
    X, lens = p.store.newest(p.config.refit_sample_cap)
    obs = np.flatnonzero(kinds == 1)
    assert np.array_equal(X, z["vector"][obs[-len(X):]]) and np.array_equal(lens, z["length"][obs[-len(X):]])
    assert p.store.inexact_count() == 0


def test_reference_engine_with_gpu_predictor_identical_report():
    if refsim.import_servesim() is None:
        pytest.skip("reference package not importable here")
    import importlib.util
    import sys
    spec = importlib.util.spec_from_file_location("record_pred_calls",
                                                  os.path.join(GOLDEN, "record_pred_calls.py"))
    rec = importlib.util.module_from_spec(spec)
    sys.modules["record_pred_calls"] = rec
    spec.loader.exec_module(rec)
    from servesim import simcore
    z = np.load(os.path.join(GOLDEN, "simcore_pred_calls.npz"))
    cfg = rec.config()
    _, ours = _predictor(cfg.run.max_len, threads=int(z["blas_threads"]))
    report = simcore.run(rec.trace(), "speculative", cfg, seed=0, predictor_override=ours)
    assert report.to_json() == str(z["report"])
