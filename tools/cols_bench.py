"""Column-kind quantize kernels (channel / head), many repetitions: per-launch times
(min / median / max) of one 1 GiB Llama-2-7B job, cluster kernel vs two-pass kernel
(ALISE_COLS_CL read once per process, so each variant runs in its own process)."""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2410_23537_b200 import kvmanager as km  # noqa: E402
from harness import synthetic  # noqa: E402

res = []
for kind, bits, packed in [("channel", 8, False), ("head", 8, False), ("channel", 4, True)]:
    lay = km.KVLayout(32, 2048, 4096, 128, kind=kind, group=128, bits=bits, packed=packed, planes_per_chunk=64)
    g = lay.geometry()
    kv = synthetic.kv_job_torch(32, 2048, 4096, seed=0, job=1, group=64)
    slab = torch.empty(g["slab_bytes"], dtype=torch.uint8, device="cuda")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    d = lay.desc()
    st = km._lib.stream_ptr()
    ts = []
    for i in range(33):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        km._lib.call("alise_kv_quantize", km._lib.C.byref(d), km._lib.ptr(kv), km._lib.ptr(slab),
                     km._lib.ptr(flag), st)
        e1.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1))
    alg = lay.elements * 2 + g["slab_bytes"]
    r = {"kind": kind, "bits": bits, "cl": os.environ.get("ALISE_COLS_CL", "1"),
         "ms_min": min(ts), "ms_med": statistics.median(ts), "ms_max": max(ts),
         "GBs_med": alg / statistics.median(ts) / 1e6}
    res.append(r)
    print(json.dumps(r), flush=True)
