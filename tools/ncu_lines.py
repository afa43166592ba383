"""Aggregate an ncu `--page source --csv --print-source cuda,sass` export per CUDA
source line: share of executed warp instructions and of warp-stall samples."""
import collections
import csv
import sys


def num(s):
    try:
        return float(s)
    except ValueError:
        return 0.0


def main(path, top=45):
    agg = collections.OrderedDict()
    fname = cur = None
    for r in csv.reader(open(path)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name", "Line No") or not r[0]:
            continue
        cur = (fname, int(r[0]), r[1].strip()[:90])
        a = agg.setdefault(cur, [0.0, 0.0])
        a[0] += num(r[7])
        a[1] += num(r[4])
    tot = sum(v[0] for v in agg.values()) or 1
    ts = sum(v[1] for v in agg.values()) or 1
    print(f"total warp instructions {tot:.0f}, stall samples {ts:.0f}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{v[0] / tot * 100:5.1f}% inst {v[1] / ts * 100:5.1f}% stall  {k[0]}:{k[1]} {k[2]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 45)
