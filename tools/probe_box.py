"""One-off probe of a GPU box: host cores/RAM, GPU topology, pinned host-link
bandwidth (D2H/H2D, each alone and both concurrently) and fp64 throughput.
Writes gpurun_out/probe_box.json."""
import json, os, subprocess, time
import torch

out = {}
def sh(c):
    try:
        return subprocess.run(c, shell=True, capture_output=True, text=True, timeout=60).stdout
    except Exception as e:
        return str(e)
out["nproc"] = os.cpu_count()
out["sched_affinity"] = len(os.sched_getaffinity(0))
out["meminfo"] = sh("head -3 /proc/meminfo")
out["lscpu"] = sh("lscpu | head -20")
out["nvidia_smi"] = sh("nvidia-smi --query-gpu=index,name,pci.bus_id,memory.total,clocks.max.sm --format=csv")
out["topo"] = sh("nvidia-smi topo -m")
out["pcie"] = sh("nvidia-smi --query-gpu=pcie.link.gen.current,pcie.link.gen.max,pcie.link.width.current --format=csv")
out["ulimit_l"] = sh("ulimit -l")
dev = torch.device("cuda:0")
res = {}
for mib in (64, 512, 2048):
    n = mib << 20
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    s1 = torch.cuda.Stream(); s2 = torch.cuda.Stream()
    for _ in range(2):
        h.copy_(d, non_blocking=True); d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    def timeit(fn, reps=5):
        torch.cuda.synchronize(); t = time.perf_counter()
        for _ in range(reps): fn()
        torch.cuda.synchronize(); return (time.perf_counter() - t) / reps
    d2h = timeit(lambda: h.copy_(d, non_blocking=True))
    h2d = timeit(lambda: d.copy_(h, non_blocking=True))
    d2 = torch.empty_like(d); h2 = torch.empty_like(h)
    def both():
        with torch.cuda.stream(s1): h.copy_(d, non_blocking=True)
        with torch.cuda.stream(s2): d2.copy_(h2, non_blocking=True)
    tb = timeit(both)
    res[mib] = {"d2h_GBs": n / d2h / 1e9, "h2d_GBs": n / h2d / 1e9, "duplex_each_GBs": n / tb / 1e9}
    del d, h, d2, h2
out["hostlink"] = res
# big pinned allocation test
try:
    t = time.perf_counter(); big = torch.empty(34 << 30, dtype=torch.uint8, pin_memory=True)
    out["pin_34GiB_s"] = time.perf_counter() - t; del big
except Exception as e:
    out["pin_34GiB_err"] = str(e)[:200]
# fp64 throughput
a = torch.randn(8192, 8192, dtype=torch.float64, device=dev)
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(3): c = a @ a
torch.cuda.synchronize(); out["dgemm_TFs"] = 3 * 2 * 8192**3 / (time.perf_counter() - t) / 1e12
out["free_mem_GiB"] = torch.cuda.mem_get_info()[0] / 2**30
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe_box.json", "w"), indent=1)
print(json.dumps(out["hostlink"]), out.get("pin_34GiB_s"), out["nproc"], out["dgemm_TFs"])
