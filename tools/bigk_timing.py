"""top_k > 16 search time (CUDA-core coarse pass + exact select) on the C4 DB."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2410_23537_b200 import predictor as pr  # noqa: E402
from harness import synthetic  # noqa: E402

db, lens = synthetic.predictor_db(1000000, 768, seed=0, dup_groups=1000)
st = pr.VectorStore(768, 1000000, dtype=np.float32)
st.add_batch(db, lens)
for B, k in ((1, 8), (1, 32), (64, 32), (1, 256), (1, 1024), (4096, 8), (4096, 32)):
    Q = torch.from_numpy(synthetic.predictor_queries(db, B, seed=1)).cuda()
    st.search_batch(Q, k)
    torch.cuda.synchronize()
    t = time.perf_counter()
    st.search_batch(Q, k)
    torch.cuda.synchronize()
    print(f"B={B} k={k}: {(time.perf_counter() - t) * 1e3:.3f} ms")
