"""Per-shard exact rescoring with and without the all-reduced global bound (one GPU
stand-in for an 8-GPU sharded search): shard = every 8th row of the C4 DB; the global
bound is the full-DB scan's bound (the max over the shards' bounds is at most that)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2410_23537_b200 import _lib  # noqa: E402
from paper_2410_23537_b200 import predictor as pr  # noqa: E402
from harness import synthetic  # noqa: E402

N, D, B, K, G = 1_000_000, 768, 4096, 8, 8
db, lens = synthetic.predictor_db(N, D, seed=0, dup_groups=1000)
full = pr.VectorStore(D, N, dtype=np.float32)
full.add_batch(db, lens)
shard = pr.VectorStore(D, N // G, dtype=np.float32)
shard.add_batch(db[::G], lens[::G])
Q = torch.from_numpy(synthetic.predictor_queries(db, B, seed=1)).cuda()
outs = [torch.empty((B, K), dtype=torch.float64, device="cuda"), torch.empty((B, K), dtype=torch.int64, device="cuda"),
        torch.empty((B, K), dtype=torch.int32, device="cuda"), torch.empty(B, dtype=torch.int32, device="cuda")]
gb = torch.empty(B, dtype=torch.float32, device="cuda")
lb = torch.empty(B, dtype=torch.float32, device="cuda")
_lib.call("alise_db_topk_scan", full._h, _lib.ptr(Q), B, K, _lib.ptr(gb), _lib.stream_ptr())
res = {}
for name, ext in (("local_only", None), ("global_bound", gb)):
    ts = []
    for rep in range(6):
        _lib.call("alise_db_topk_scan", shard._h, _lib.ptr(Q), B, K, _lib.ptr(lb), _lib.stream_ptr())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.call("alise_db_topk_rescore", shard._h, _lib.ptr(Q), B, K, _lib.ptr(ext), *[_lib.ptr(t) for t in outs],
                  _lib.stream_ptr())
        e1.record()
        torch.cuda.synchronize()
        if rep:
            ts.append(e0.elapsed_time(e1))
    res[name] = {"rescore_ms": sum(ts) / len(ts), "mean_count": float(outs[3].float().mean())}
print(json.dumps(res))
