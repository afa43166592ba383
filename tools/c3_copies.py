"""Raw duplex pinned-copy rate for the C3 transfer sizes (one slab per job, ShareGPT
mix), to separate the host link's small-copy efficiency from the swap pipeline's."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2410_23537_b200 import kvmanager as km  # noqa: E402
from harness import synthetic  # noqa: E402

ctx = synthetic.sharegpt_job_tokens(256, seed=0)
sizes = [km.KVLayout(32, int(t), 4096, 128, kind="rows", group=64, bits=4, packed=True).geometry()["slab_bytes"]
         for t in ctx]
mx = max(sizes)
dev = [torch.empty(mx, dtype=torch.uint8, device="cuda") for _ in range(2)]
host = [torch.empty(mx, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
s_out, s_in = torch.cuda.Stream(), torch.cuda.Stream()


def run():
    for i, n in enumerate(sizes):
        with torch.cuda.stream(s_out):
            host[0][:n].copy_(dev[0][:n], non_blocking=True)
        with torch.cuda.stream(s_in):
            dev[1][:sizes[i - 1]].copy_(host[1][:sizes[i - 1]], non_blocking=True)
    torch.cuda.synchronize()


run()
t = time.perf_counter()
for _ in range(3):
    run()
dt = (time.perf_counter() - t) / 3
total = 2 * sum(sizes)
print(json.dumps({"jobs": len(sizes), "mean_MB": sum(sizes) / len(sizes) / 1e6, "duplex_GBs": total / dt / 1e9}))
