"""Small-shape workload for compute-sanitizer (memcheck / racecheck / synccheck): every
hot kernel once -- KV quantize+offload and upload+dequantize for the rows (g=128 INT8,
g=64 INT4 packed, absmax), channel and head kinds (single-pass cluster kernel and the
two-pass fallback), the drop-in quantize/dequantize (float64 rows), and the predictor
scan (tcgen05, small and large batch paths), exact rescoring, exhaustive path and finish.
Results are checked against the oracle so a sanitizer run also proves the outputs."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from harness import parity, synthetic  # noqa: E402
from oracle import kv_oracle, pred_oracle  # noqa: E402
from paper_2410_23537_b200 import kvmanager as km  # noqa: E402
from paper_2410_23537_b200 import predictor as pr  # noqa: E402

torch.cuda.set_device(0)
bad = 0
# ---- KV data plane
L, T, H = 2, 96, 512
for kind, group, bits, packed, mode in [("rows", 128, 8, False, "asymmetric"), ("rows", 64, 4, True, "asymmetric"),
                                        ("rows", 64, 8, False, "absmax"), ("channel", 128, 8, False, "asymmetric"),
                                        ("head", 128, 4, True, "asymmetric")]:
    lay = km.KVLayout(L, T, H, 128, kind=kind, group=group, bits=bits, packed=packed, mode=mode)
    kv = synthetic.kv_job_torch(L, T, H, seed=1, job=2, group=64)
    g = lay.geometry()
    pool = km.HostSlabPool(g["slab_bytes"] + 4096)
    eng = km.KVSwapEngine()
    addr = pool.alloc(g["slab_bytes"])
    eng.offload(lay, kv, addr)
    out = torch.zeros_like(kv)
    eng.upload(lay, addr, out)
    torch.cuda.synchronize()
    planes, _v, b = parity.kv_check_planes(lay, kv.cpu().numpy(), pool.view(addr, g["slab_bytes"]), out.cpu().numpy())
    bad += len(b)
    print(kind, group, bits, packed, mode, "planes", planes, "mismatches", len(b))
    eng.close()
    pool.close()
os.environ["ALISE_COLS_TWOPASS"] = "1"  # read once per call: the two-pass column kernel
x = np.random.default_rng(0).standard_normal((40, 200)) * 3.0
qt = km.quantize(x, 8)
c, s, z = kv_oracle.quantize_rows(x, 8)
bad += int(not (np.array_equal(qt.values, c) and np.array_equal(qt.scale, s) and np.array_equal(km.dequantize(qt),
                                                                                         kv_oracle.dequantize_rows(c, s, z))))
# ---- predictor
n, d = 3000, 256
rng = np.random.default_rng(3)
db = rng.standard_normal((n, d)).astype(np.float32)
db /= np.linalg.norm(db, axis=1, keepdims=True)
db[100:140] = db[7]  # ties
lens = rng.integers(1, 2048, size=n).astype(np.int32)
store = pr.VectorStore(d, 4096, dtype=np.float32)
store.add_batch(db, lens)
for B in (8, 600):
    Q = db[rng.integers(0, n, size=B)] + 0.05 * rng.standard_normal((B, d)).astype(np.float32)
    Q = (Q / np.linalg.norm(Q, axis=1, keepdims=True)).astype(np.float32)
    sims, seqs, _l, _c, _ = store.search_batch(Q, 8)
    torch.cuda.synchronize()
    for i in range(0, B, max(1, B // 16)):
        es, _el, eq = pred_oracle.search_exact(db, lens, np.arange(n), Q[i], 8)
        bad += int(not np.array_equal(seqs[i].cpu().numpy(), eq))
    reg = pr.FallbackRegressor(d, 32, seed=0)
    p = pr.LengthPredictor(pr.PredictorConfig(dimension=d, db_capacity=4096), regressor=reg, store=store)
    o, r = p.predict_batch(Q)
    rl, rr = pred_oracle.predict_batch(db, lens, np.arange(n), Q, reg.w1, reg.b1, reg.w2, reg.b2)
    bad += int(not np.array_equal(o.cpu().numpy(), rl))
    print("predictor B", B, "ok" if not bad else "MISMATCH")
# top_k above 16 (single-query and batched CUDA-core coarse passes + exact select)
for B, k in ((1, 40), (24, 40), (6, 300)):
    Q = db[rng.integers(0, n, size=B)] + 0.05 * rng.standard_normal((B, d)).astype(np.float32)
    Q = (Q / np.linalg.norm(Q, axis=1, keepdims=True)).astype(np.float32)
    sims, seqs, _l, _c, _ = store.search_batch(Q, k)
    torch.cuda.synchronize()
    for i in range(B):
        es, _el, eq = pred_oracle.search_exact(db, lens, np.arange(n), Q[i], k)
        bad += int(not np.array_equal(seqs[i].cpu().numpy()[:len(eq)], eq))
    print("top-k", k, "B", B, "ok" if not bad else "MISMATCH")
torch.cuda.synchronize()
print("sanitize workload mismatches", bad)
sys.exit(1 if bad else 0)
