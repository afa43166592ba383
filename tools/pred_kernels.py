"""Per-kernel device time of LengthPredictor.predict_batch on the C4 DB (1M x 768),
warm caches, measured in-process with CUPTI (torch.profiler).
usage: python tools/pred_kernels.py [N] [B,B,...]"""
import collections
import json
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
from paper_2410_23537_b200 import predictor as pr  # noqa: E402
from harness import synthetic  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
BS = [int(b) for b in sys.argv[2].split(",")] if len(sys.argv) > 2 else [256, 64, 1]
D = 768
db, lens = synthetic.predictor_db(N, D, seed=0, dup_groups=1000)
store = pr.VectorStore(D, N, dtype=np.float32)
store.add_batch(db, lens)
reg = pr.FallbackRegressor(D, 32, seed=0)
reg.b2 = 5.0
p = pr.LengthPredictor(pr.PredictorConfig(dimension=D, db_capacity=N), regressor=reg, store=store)
for B in BS:
    Q = torch.from_numpy(synthetic.predictor_queries(db, B, seed=1)).cuda()
    for _ in range(3):
        p.predict_batch(Q)
    torch.cuda.synchronize()
    reps = 10
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(reps):
            p.predict_batch(Q)
        torch.cuda.synchronize()
    agg = collections.defaultdict(float)
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            agg[ev.name.split("(")[0][:60]] += ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
    tot = sum(agg.values())
    out = {"B": B, "total_us_per_call": tot / reps,
           "kernels_us": {k: round(v / reps, 2) for k, v in sorted(agg.items(), key=lambda x: -x[1])}}
    print(json.dumps(out), flush=True)
