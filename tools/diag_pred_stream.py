"""Diagnose the reference predictor call-stream replay: print the first mismatches with
the GPU top-k, the numpy (reference-arithmetic) top-k over the same store contents and
both MLP outputs."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2410_23537_b200 import predictor as pr  # noqa: E402

z = np.load(os.path.join(ROOT, "tests/golden/simcore_pred_calls.npz"))
cfg = pr.PredictorConfig(max_len=int(z["max_len"]))
from oracle import pred_oracle as po  # noqa: E402
ORDER = sys.argv[1] if len(sys.argv) > 1 else "blas"
p = pr.LengthPredictor(cfg, store=pr.VectorStore(cfg.dimension, cfg.db_capacity, order=ORDER,
                                                 blas_threads=int(z["blas_threads"])))
kinds, offs, toks = z["kind"], z["offsets"], z["tokens"]
shown = 0
for i, kind in enumerate(kinds):
    if kind == 0:
        tokens = toks[offs[i]:offs[i + 1]].tolist()
        n, prov, vec = p.predict(tokens, int(z["request_id"][i]))
        want = (int(z["length"][i]), pr.RETRIEVED if z["retrieved"][i] else pr.FALLBACK)
        if (n, prov) != want:
            V, L, S = p.store.export()
            sims_all = po.blas_gemv(V, vec, int(z["blas_threads"]))
            o = np.lexsort((S, -sims_all))[:8]
            s_np, l_np, q_np = sims_all[o], L[o], S[o]
            g = p.store.search(vec, 8)
            print(f"call {i}: got {(n, prov)} want {want}; vec equal {np.array_equal(vec, z['vector'][i])}; "
                  f"store size {p.store.size}")
            print("  gpu sims", np.array(g[0]).tolist(), "lens", np.array(g[1]).tolist())
            print("  gpu seqs", np.array(g[2]).tolist())
            print("  ora sims", np.array(s_np).tolist(), "lens", l_np.tolist(), "seqs", q_np.tolist())
            print("  mlp host", p.regressor.predict_len.__doc__ is None, int(round(np.exp(min(p.regressor._forward(vec[None])[1][0], np.log(cfg.max_len) + 1)))),
                  "gpu", int(p.regressor.predict_len_batch(vec[None], cfg.max_len)[0]))
            shown += 1
            if shown >= 8:
                break
    else:
        p.observe(z["vector"][i], int(z["length"][i]))
print("done; mismatches shown", shown)
