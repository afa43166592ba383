import sys
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2410_23537_b200 import predictor as pr
from harness import synthetic
db, lens = synthetic.predictor_db(1000000, 768, seed=0, dup_groups=1000)
st = pr.VectorStore(768, 1000000, dtype=np.float32); st.add_batch(db, lens)
Q = torch.from_numpy(synthetic.predictor_queries(db, 1, seed=1)).cuda()
for _ in range(2):
    st.search_batch(Q, 32)
torch.cuda.synchronize()
