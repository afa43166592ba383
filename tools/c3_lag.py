"""C3 swap pipeline (256 ShareGPT-mix jobs, INT4 g=64 packed) with different
offload/upload lags: fp16 GB/s and link utilisation."""
import json
import sys

sys.path.insert(0, ".")
sys.argv = ["bench.py"]
import bench  # noqa: E402
from paper_2410_23537_b200 import kvmanager as km  # noqa: E402
from harness import synthetic  # noqa: E402

args = bench.parse()
args.steps, args.warmup = 2, 1
links = bench.link_peaks(0)
ctx = synthetic.sharegpt_job_tokens(256, seed=0)
lays = [km.KVLayout(args.layers, int(t), args.hidden, args.head_dim, kind="rows", group=64, bits=4, packed=True)
        for t in ctx]
for hs, lag in ((4, 1), (8, 1), (8, 3), (16, 4)):
    args.host_slabs, args.lag = hs, lag
    r = bench.kv_bench(args, 1, 0, 0, layouts=lays, e2e=False)
    print(json.dumps({"host_slabs": hs, "lag": lag, "GBs": round(r["value"], 1), "link": round(r["link_GBs_total"], 1),
                      "link_frac": round(r["link_GBs_total"] / links["duplex_total_GBs"], 3)}), flush=True)
