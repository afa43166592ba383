"""B = 1 predict_batch calls on the C4 DB (for the ALISE_FINISH_TIMING build of k_finish:
per-phase clock64 cycles of the finish kernel)."""
import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2410_23537_b200 import predictor as pr
from harness import synthetic
N, D = 1000000, 768
db, lens = synthetic.predictor_db(N, D, seed=0, dup_groups=1000)
st = pr.VectorStore(D, N, dtype=np.float32); st.add_batch(db, lens)
reg = pr.FallbackRegressor(D, 32, seed=0); reg.b2 = 5.0
p = pr.LengthPredictor(pr.PredictorConfig(dimension=D, db_capacity=N), regressor=reg, store=st)
g = np.random.default_rng(3)
q = g.standard_normal((1, D)).astype(np.float32); q /= np.linalg.norm(q)
for _ in range(4):
    p.predict_batch(q); torch.cuda.synchronize()
