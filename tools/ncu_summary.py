"""Summarise an ncu --set full report (one kernel launch) into a short text file.
usage: python tools/ncu_summary.py report.ncu-rep out.txt [algorithmic_bytes]"""
import csv
import io
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
alg = float(sys.argv[3]) if len(sys.argv) > 3 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
keys = ["Kernel Name", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "lts__t_bytes.sum", "l1tex__t_bytes.sum"]
with open(out, "w") as f:
    f.write(f"ncu --set full --clock-control none report: {rep}\n")
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        for k in keys:
            if k in d:
                f.write(f"  {k:62s} {d[k]} {u.get(k, '')}\n")
        try:
            t_ns = float(d["gpu__time_duration.sum"]) * (1e3 if u["gpu__time_duration.sum"] == "us" else 1)
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rd = float(d["dram__bytes_read.sum"]) * scale.get(u["dram__bytes_read.sum"], 1)
            wr = float(d["dram__bytes_write.sum"]) * scale.get(u["dram__bytes_write.sum"], 1)
            f.write(f"  traffic (dram read+write) = {rd + wr:.4g} B ; dram GB/s = {(rd + wr) / t_ns:.1f}\n")
            if alg:
                f.write(f"  algorithmic bytes = {alg:.4g} B ; traffic/algorithmic = {(rd + wr) / alg:.3f} ;"
                        f" algorithmic GB/s under ncu = {alg / t_ns:.1f}\n")
        except Exception as e:  # noqa: BLE001
            f.write(f"  (traffic summary unavailable: {e})\n")
print(open(out).read())
