"""Replay the recorded predictor stream up to a call index, then search the grown store
and a freshly built copy of it (both orders) to localise state-dependent differences."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2410_23537_b200 import predictor as pr  # noqa: E402

z = np.load(os.path.join(ROOT, "tests/golden/simcore_pred_calls.npz"))
stop = int(sys.argv[1]) if len(sys.argv) > 1 else 1035
cfg = pr.PredictorConfig(max_len=int(z["max_len"]))
p = pr.LengthPredictor(cfg, store=pr.VectorStore(cfg.dimension, cfg.db_capacity, order="blas", blas_threads=8))
kinds, offs, toks = z["kind"], z["offsets"], z["tokens"]
for i in range(stop):
    if kinds[i] == 0:
        p.predict(toks[offs[i]:offs[i + 1]].tolist(), int(z["request_id"][i]))
    else:
        p.observe(z["vector"][i], int(z["length"][i]))
vec = p.embed(toks[offs[stop]:offs[stop + 1]].tolist())
V, L, S = p.store.export()
for order in ("blas", "exact"):
    p.store.set_order(order, 8)
    s, q, l_, c, _ = p.store.search_batch(vec[None], 8)
    torch.cuda.synchronize()
    print(order, "grown ", int(c[0]), q[0].cpu().numpy().tolist())
    fresh = pr.VectorStore(cfg.dimension, cfg.db_capacity, order=order, blas_threads=8)
    fresh.add_batch(V[np.argsort(S)], L[np.argsort(S)])
    s2, q2, l2, c2, _ = fresh.search_batch(vec[None], 8)
    torch.cuda.synchronize()
    print(order, "fresh ", int(c2[0]), q2[0].cpu().numpy().tolist())
import ctypes  # noqa: E402
os.environ["ALISE_SCAN_STATS"] = "1"
