"""Does a KV quantize launch run slower on a buffer it has not touched recently?  One
Llama-2-7B job (1 GiB fp16) per launch, INT8 g=128 rows; per-launch CUDA events.
  same      : one buffer, back to back
  rr        : round robin over NB distinct buffers, back to back
  same_idle : one buffer, ~2 ms of idle GPU before each launch (the swap step's gating)
  rr_idle   : NB buffers round robin, idle before each launch
  rr_touch  : as rr_idle, plus a strided read of the next buffer (one element per
              64 KiB of source and slab) just before its launch"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2410_23537_b200 import kvmanager as km  # noqa: E402
from harness import synthetic  # noqa: E402

NB = int(sys.argv[1]) if len(sys.argv) > 1 else 16
lay = km.KVLayout(32, 2048, 4096, 128, kind="rows", group=128, bits=8, packed=False, planes_per_chunk=64)
g = lay.geometry()
base = synthetic.kv_job_torch(32, 2048, 4096, seed=0, job=1, group=128)
kvs = [base] + [base.clone() for _ in range(NB - 1)]
slabs = [torch.empty(g["slab_bytes"], dtype=torch.uint8, device="cuda") for _ in range(NB)]
flag = torch.zeros(1, dtype=torch.int32, device="cuda")
d = lay.desc()
st = km._lib.stream_ptr()
alg = lay.elements * 2 + g["slab_bytes"]


def q(i):
    km._lib.call("alise_kv_quantize", km._lib.C.byref(d), km._lib.ptr(kvs[i]), km._lib.ptr(slabs[i]),
                 km._lib.ptr(flag), st)


def touch(i):
    kvs[i].view(-1)[::32768].float().sum()
    slabs[i][::65536].sum()


def run(mode, n=32):
    ts = []
    for r in range(n):
        i = 0 if mode.startswith("same") else r % NB
        if "idle" in mode or "touch" in mode:
            torch.cuda._sleep(2_000_000)
        if "touch" in mode:
            touch(i)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        q(i)
        e1.record()
        ts.append((e0, e1))
    torch.cuda.synchronize()
    ms = sorted(a.elapsed_time(b) for a, b in ts)
    med = ms[len(ms) // 2]
    return {"mode": mode, "median_ms": round(med, 4), "GBs": round(alg / med / 1e6, 1),
            "min_ms": round(ms[0], 4), "max_ms": round(ms[-1], 4)}


for i in range(NB):
    q(i)
torch.cuda.synchronize()
for mode in ("same", "rr", "same_idle", "rr_idle", "rr_touch", "same", "rr", "rr_idle"):
    print(json.dumps(run(mode)), flush=True)
