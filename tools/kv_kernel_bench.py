"""Device-to-device timing of the KV quantize / dequantize kernels alone (one
Llama-2-7B job per launch, 1 GiB fp16), CUDA events, after warm-up."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2410_23537_b200 import kvmanager as km  # noqa: E402
from harness import synthetic  # noqa: E402

CASES = [("rows", 128, 8, False), ("rows", 64, 4, True), ("rows", 64, 8, False),
         ("channel", 0, 8, False), ("head", 0, 8, False)]
if len(sys.argv) > 1:  # e.g. "rows:128:8:0,rows:64:4:1"
    CASES = [(k, int(g), int(b), bool(int(p))) for k, g, b, p in (c.split(":") for c in sys.argv[1].split(","))]
res = []
for kind, group, bits, packed in CASES:
    lay = km.KVLayout(32, 2048, 4096, 128, kind=kind, group=group or 128, bits=bits, packed=packed,
                      planes_per_chunk=64)
    g = lay.geometry()
    kv = synthetic.kv_job_torch(32, 2048, 4096, seed=0, job=1, group=group or 64)
    slab = torch.empty(g["slab_bytes"], dtype=torch.uint8, device="cuda")
    out = torch.empty_like(kv)
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    d = lay.desc()
    st = km._lib.stream_ptr()

    def q():
        km._lib.call("alise_kv_quantize", km._lib.C.byref(d), km._lib.ptr(kv), km._lib.ptr(slab),
                     km._lib.ptr(flag), st)

    def dq():
        km._lib.call("alise_kv_dequantize", km._lib.C.byref(d), km._lib.ptr(slab), km._lib.ptr(out), st)

    for fn in (q, dq):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
    # median of 5 rounds of 10 back-to-back launches (single rounds vary by ~10-20% between boxes)
    qs, ds = [], []
    for _ in range(5):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        reps = 10
        e[0].record()
        for _ in range(reps):
            q()
        e[1].record()
        for _ in range(reps):
            dq()
        e[2].record()
        torch.cuda.synchronize()
        qs.append(e[0].elapsed_time(e[1]) / reps)
        ds.append(e[1].elapsed_time(e[2]) / reps)
    n = lay.elements
    alg = n * 2 + g["slab_bytes"]
    qms = sorted(qs)[2]
    dms = sorted(ds)[2]
    r = {"kind": kind, "group": group, "bits": bits, "packed": packed, "slab_bytes": g["slab_bytes"],
         "quant_ms": qms, "quant_GBs": alg / qms / 1e6, "dequant_ms": dms, "dequant_GBs": alg / dms / 1e6,
         "exact_roundtrip_err_ok": None}
    res.append(r)
    print(json.dumps(r))
    del kv, slab, out
    torch.cuda.empty_cache()
import os  # noqa: E402
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/kv_kernels%s.json" % os.environ.get("ALISE_QTILE", ""), "w"), indent=1)
