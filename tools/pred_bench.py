"""Time the predictor hot path at BASELINE config 4 (1M x 768 DB, B queries)."""
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
t = time.time()
db, lens = synthetic.predictor_db(N, D, seed=0, dup_groups=1000)
store = pr.VectorStore(D, N, dtype=np.float32)
store.add_batch(db, lens)
torch.cuda.synchronize()
print("db build s", time.time() - t, flush=True)
reg = pr.FallbackRegressor(D, 32, seed=0)
reg.b2 = 5.0
p = pr.LengthPredictor(pr.PredictorConfig(dimension=D, db_capacity=N), regressor=reg, store=store)
res = []
BS = [int(b) for b in sys.argv[2].split(",")] if len(sys.argv) > 2 else [4096, 1024, 256, 64, 1]
for B in BS:
    Q = torch.from_numpy(synthetic.predictor_queries(db, B, seed=1)).cuda()
    for _ in range(3):
        p.predict_batch(Q)
    torch.cuda.synchronize()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    reps = 5 if B >= 1024 else 20
    e0.record()
    for _ in range(reps):
        store.search_batch(Q, 8)
    e1.record()
    for _ in range(reps):
        p.predict_batch(Q)
    e2.record()
    torch.cuda.synchronize()
    ms_s = e0.elapsed_time(e1) / reps
    ms_p = e1.elapsed_time(e2) / reps
    flops = 2.0 * B * N * D
    r = {"B": B, "N": N, "search_ms": ms_s, "predict_ms": ms_p, "qps": B / ms_p * 1e3,
         "coarse_TFLOPs_eff": flops / ms_s / 1e9, "inexact": store.inexact_count()}
    res.append(r)
    print(json.dumps(r), flush=True)
json.dump(res, open("gpurun_out/pred_bench.json", "w"), indent=1)
