"""Timeline of C2 swap steps (nsys is not in the image: CUPTI through torch.profiler):
16 Llama-2-7B jobs x 2048 tokens, INT8 rows g=128, the bench's pipeline (offload job j
while uploading job j-1, 8 pinned host slabs).  Writes the per-engine busy time and the
overlap of the copy engines with each other and with the quantize / dequantize kernels
to gpurun_out/c2_timeline.json (+ the raw trace, gzip)."""
import gzip
import json
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
from paper_2410_23537_b200 import kvmanager as km  # noqa: E402
from harness import synthetic  # noqa: E402

J, H, LAG = 16, 8, 1
lay = km.KVLayout(32, 2048, 4096, 128, kind="rows", group=128, bits=8)
geo = lay.geometry()
kvs = [synthetic.kv_job_torch(32, 2048, 4096, seed=0, job=j, group=128) for j in range(J)]
pool = km.HostSlabPool(H * ((geo["slab_bytes"] + 255) // 256 * 256))
slabs = [pool.alloc(geo["slab_bytes"]) for _ in range(H)]
eng = km.KVSwapEngine()
ev_off = [km._Event() for _ in range(H)]
ev_up = [km._Event() for _ in range(H)]
used = [False] * H


def step():
    for j in range(J + LAG):
        if j < J:
            s = j % H
            if used[s]:
                eng.depend(ev_up[s].h)
            eng.offload(lay, kvs[j], slabs[s], event=ev_off[s].h)
        u = j - LAG
        if 0 <= u < J:
            s = u % H
            eng.depend(ev_off[s].h)
            eng.upload(lay, slabs[s], kvs[u], event=ev_up[s].h)
            used[s] = True
    torch.cuda.synchronize()


for _ in range(2):
    step()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(2):
        step()
os.makedirs("gpurun_out", exist_ok=True)
prof.export_chrome_trace("/tmp/c2_trace.json")
tr = json.load(open("/tmp/c2_trace.json"))
ev = [e for e in tr["traceEvents"] if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]


def cls(e):
    n = e["name"]
    if e["cat"] == "gpu_memcpy":
        return "d2h" if "DtoH" in n else ("h2d" if "HtoD" in n else "d2d")
    if "quant" in n and "dequant" not in n:
        return "quantize"
    if "dequant" in n or "expand" in n:
        return "dequantize"
    return "other"


iv = {}
for e in ev:
    iv.setdefault(cls(e), []).append((e["ts"], e["ts"] + e["dur"]))


def union(xs):
    xs = sorted(xs)
    out = []
    for a, b in xs:
        if out and a <= out[-1][1]:
            out[-1] = (out[-1][0], max(out[-1][1], b))
        else:
            out.append((a, b))
    return out


def length(xs):
    return sum(b - a for a, b in xs)


def inter(a, b):
    i = j = 0
    out = []
    while i < len(a) and j < len(b):
        lo, hi = max(a[i][0], b[j][0]), min(a[i][1], b[j][1])
        if lo < hi:
            out.append((lo, hi))
        if a[i][1] < b[j][1]:
            i += 1
        else:
            j += 1
    return out


U = {k: union(v) for k, v in iv.items()}
t0 = min(a for v in U.values() for a, _ in v)
t1 = max(b for v in U.values() for _, b in v)
span = t1 - t0
kern = union(U.get("quantize", []) + U.get("dequantize", []))
both = inter(U.get("d2h", []), U.get("h2d", []))
res = {"workload": f"2 C2 steps of {J} jobs (INT8 rows g=128, {geo['n_chunks']} chunks/job), lag {LAG}, {H} slabs",
       "span_us": span,
       "busy_us": {k: length(v) for k, v in U.items()},
       "busy_frac": {k: length(v) / span for k, v in U.items()},
       "both_copy_directions_busy_frac": length(both) / span,
       "kernels_overlapped_by_copies_frac": length(inter(kern, union(U.get("d2h", []) + U.get("h2d", [])))) / max(1, length(kern)),
       "copy_bytes": 2 * 2 * J * geo["slab_bytes"],
       "link_GBs_over_span": 2 * 2 * J * geo["slab_bytes"] / (span * 1e3)}
json.dump(res, open("gpurun_out/c2_timeline.json", "w"), indent=1)
with gzip.open("gpurun_out/c2_trace.json.gz", "wt") as f:
    json.dump({"traceEvents": ev}, f)
print(json.dumps(res))
eng.close()
pool.close()
