"""A few predict_batch calls on an N-row slice of the C4 DB (for ncu captures of the
scan at shard sizes).   usage: python tools/scan_one.py N B"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2410_23537_b200 import predictor as pr  # noqa: E402
from harness import synthetic  # noqa: E402

N, B = int(sys.argv[1]), int(sys.argv[2])
db, lens = synthetic.predictor_db(N, 768, seed=0, dup_groups=1000)
st = pr.VectorStore(768, N, dtype=np.float32)
st.add_batch(db, lens)
Q = torch.from_numpy(synthetic.predictor_queries(db, B, seed=1)).cuda()
for _ in range(3):
    st.search_batch(Q, 8)
torch.cuda.synchronize()
