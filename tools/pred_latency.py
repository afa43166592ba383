"""Per-request latency of the drop-in predictor API (predict_vector: host vector in,
(length, provenance) out) on the C4 DB (1M x 768)."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2410_23537_b200 import predictor as pr  # noqa: E402
from harness import synthetic  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
D = 768
db, lens = synthetic.predictor_db(N, D, seed=0, dup_groups=1000)
store = pr.VectorStore(D, N, dtype=np.float32)
store.add_batch(db, lens)
reg = pr.FallbackRegressor(D, 32, seed=0)
reg.b2 = 5.0
p = pr.LengthPredictor(pr.PredictorConfig(dimension=D, db_capacity=N), regressor=reg, store=store)
Q = synthetic.predictor_queries(db, 64, seed=1).astype(np.float64)
for i in range(5):
    p.predict_vector(Q[i])
torch.cuda.synchronize()
ts = []
for i in range(64):
    t0 = time.perf_counter()
    p.predict_vector(Q[i])
    ts.append(time.perf_counter() - t0)
ts.sort()
print(json.dumps({"api": "LengthPredictor.predict_vector", "N": N, "p50_ms": ts[32] * 1e3, "p90_ms": ts[57] * 1e3,
                  "min_ms": ts[0] * 1e3}))
p.enable_graphs()
ref = [p.predict_vector(Q[i]) for i in range(64)]
ts = []
for i in range(64):
    t0 = time.perf_counter()
    r = p.predict_vector(Q[i])
    ts.append(time.perf_counter() - t0)
    assert r == ref[i]
ts.sort()
print(json.dumps({"api": "LengthPredictor.predict_vector (CUDA graph)", "N": N, "p50_ms": ts[32] * 1e3,
                  "p90_ms": ts[57] * 1e3, "min_ms": ts[0] * 1e3}))
