"""In-step quantize kernel time with and without the upload direction running: the C2
swap pipeline offloads 8 Llama-2-7B jobs (INT8 g=128) to pinned host slabs, (a) alone,
(b) with the previous job's upload + dequantize running concurrently (as in bench.py).
Prints the average quantize chunk launch time and its HBM GB/s for both."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2410_23537_b200 import kvmanager as km  # noqa: E402
from harness import synthetic  # noqa: E402

J, H = 8, 8
PPC = int(sys.argv[1]) if len(sys.argv) > 1 else 0  # planes per transfer chunk (0: default)
lay = km.KVLayout(32, 2048, 4096, 128, kind="rows", group=128, bits=8, planes_per_chunk=PPC)
geo = lay.geometry()
pool = km.HostSlabPool(H * ((geo["slab_bytes"] + 255) // 256 * 256))
slabs = [pool.alloc(geo["slab_bytes"]) for _ in range(H)]
kvs = [synthetic.kv_job_torch(32, 2048, 4096, seed=0, job=j, group=128, device="cuda") for j in range(J)]
eng = km.KVSwapEngine(device=0)
hp = torch.cuda.Stream(priority=-1)
out = {}
# keep-alive probe: a low-priority stream keeps one SM spinning during the pipeline, so
# the GPU never idles between the link-gated quantize chunks (clock/power-state test)
lo = torch.cuda.Stream(priority=0)
spin = torch.empty(1, device="cuda")
for mode in ("offload_only", "offload_with_upload", "offload_only_keepalive"):
    with torch.cuda.stream(hp):
        for rep in range(2):
            eng.kernel_stats()
            eng.set_timing(rep == 1)
            evs = [km._Event() for _ in range(J)]
            if mode.endswith("keepalive"):
                with torch.cuda.stream(lo):
                    torch.cuda._sleep(int(2e9))  # ~1 s of spinning on one SM
            for j in range(J):
                eng.offload(lay, kvs[j], slabs[j % H], event=evs[j].h)
                if mode == "offload_with_upload" and j > 0:
                    eng.depend(evs[j - 1].h)  # the upload reads what offload j-1 wrote
                    eng.upload(lay, slabs[(j - 1) % H], kvs[j - 1])
            torch.cuda.synchronize()
    eng.set_timing(False)
    qms, qn, dms, dn = eng.kernel_stats()
    job_bytes = lay.elements * 2 + geo["slab_bytes"]  # algorithmic bytes of one job's quantize
    out[mode] = {"quant_launch_ms": qms / max(qn, 1), "quant_GBs": J * job_bytes / max(qms, 1e-9) / 1e6,
                 "launches": qn, "dequant_launch_ms": dms / max(dn, 1) if dn else None}
print(json.dumps(out))
