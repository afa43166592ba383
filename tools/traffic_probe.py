"""Launch exactly the bench's kernel configurations (for ncu --set full): one job's
k_quant_tile / k_dequant_wide chunk launches (default 128 MiB-code chunks, g=128,
INT8) and k_scan at C4 (B=4096 x 1M x 768).
Usage under ncu: -k regex:'k_quant_tile|k_dequant_wide|k_scan' -c 3."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2410_23537_b200 import kvmanager as km  # noqa: E402
from paper_2410_23537_b200 import predictor as pr  # noqa: E402
from harness import synthetic  # noqa: E402

lay = km.KVLayout(32, 2048, 4096, 128, kind="rows", group=128, bits=8)
kv = synthetic.kv_job_torch(32, 2048, 4096, seed=0, job=1, group=128)
g = lay.geometry()
slab = torch.empty(g["slab_bytes"], dtype=torch.uint8, device="cuda")
flag = torch.zeros(1, dtype=torch.int32, device="cuda")
km._lib.call("alise_kv_quantize", km._lib.C.byref(lay.desc()), km._lib.ptr(kv), km._lib.ptr(slab),
             km._lib.ptr(flag), km._lib.stream_ptr())
out = torch.empty_like(kv)
km._lib.call("alise_kv_dequantize", km._lib.C.byref(lay.desc()), km._lib.ptr(slab), km._lib.ptr(out),
             km._lib.stream_ptr())
torch.cuda.synchronize()
print("quant chunks", g["n_chunks"], "values per chunk", lay.elements // g["n_chunks"])
del kv, slab, out
db, lens = synthetic.predictor_db_torch(1_000_000, 768, seed=0, dup_groups=1000)
store = pr.VectorStore(768, 1_000_000, dtype=np.float32)
store.add_batch(db, lens)
Q = synthetic.predictor_queries_torch(db, 4096, seed=1)
store.search_batch(Q, 8)
torch.cuda.synchronize()
print("scan done")
