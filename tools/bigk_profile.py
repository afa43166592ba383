import sys, collections
import numpy as np, torch
from torch.profiler import ProfilerActivity, profile
sys.path.insert(0, ".")
from paper_2410_23537_b200 import predictor as pr
from harness import synthetic
db, lens = synthetic.predictor_db(1000000, 768, seed=0, dup_groups=1000)
st = pr.VectorStore(768, 1000000, dtype=np.float32); st.add_batch(db, lens)
for B, k in ((1, 32), (64, 32)):
    Q = torch.from_numpy(synthetic.predictor_queries(db, B, seed=1)).cuda()
    st.search_batch(Q, k); torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        st.search_batch(Q, k); torch.cuda.synchronize()
    agg = collections.defaultdict(float)
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            agg[ev.name.split("(")[0][:50]] += ev.device_time_total
    print(B, k, dict(agg))
