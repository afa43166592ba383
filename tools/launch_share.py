"""Summarise an `ncu --metrics gpu__time_duration.sum --csv --log-file` launch list:
per-kernel launch count, total and mean time, and share of the listed GPU time
(ncu serialises launches with cold caches: compare shares, not absolutes).
usage: python tools/launch_share.py launches.csv [out.txt] [--only REGEX]"""
import collections
import csv
import re
import sys


def short(name: str) -> str:
    m = re.match(r"(?:void\s+)?([\w:]+(?:<[^()]*>)?)", name)
    s = m.group(1) if m else name
    return s if len(s) < 90 else s[:87] + "..."


def main(argv):
    path = argv[1]
    out = argv[2] if len(argv) > 2 and not argv[2].startswith("--") else None
    only = None
    if "--only" in argv:
        only = re.compile(argv[argv.index("--only") + 1])
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0] != "ID"]
    agg = collections.OrderedDict()
    for r in rows:
        name, unit, val = r[4], r[13], float(r[14])
        ns = val * {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(unit, 1)
        if only and not only.search(name):
            continue
        a = agg.setdefault(short(name), [0, 0.0])
        a[0] += 1
        a[1] += ns
    tot = sum(v[1] for v in agg.values()) or 1
    lines = [f"launch list: {path} ({sum(v[0] for v in agg.values())} launches, {tot / 1e6:.3f} ms listed)",
             f"{'share':>6} {'launches':>8} {'total ms':>10} {'mean us':>9}  kernel"]
    for k, (n, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{ns / tot * 100:5.1f}% {n:8d} {ns / 1e6:10.3f} {ns / n / 1e3:9.1f}  {k}")
    text = "\n".join(lines) + "\n"
    if out:
        open(out, "w").write(text)
    print(text)


if __name__ == "__main__":
    main(sys.argv)
