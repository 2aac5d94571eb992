"""Warp-stall samples per (file, CUDA line) of an ncu report's source page (dev tool).

    ncu -i rep.ncu-rep --page source --csv --print-source cuda,sass > src.csv
    python tools/ncu_lines.py src.csv [top] [--ranges kernels.cu:a-b=name ...]
"""
import collections
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    top = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 30
    ranges = [a for a in sys.argv[2:] if "=" in a]
    f = hdr = cur = None
    si = 0
    agg, src = collections.Counter(), {}
    for r in rows:
        if r and r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            si = hdr.index("Warp Stall Sampling (All Samples)")
            continue
        if not hdr or len(r) < len(hdr):
            continue
        if r[0]:
            cur = (f, int(r[0]))
            src[cur] = r[1]
        try:
            agg[cur] += int(r[si] or 0)
        except ValueError:
            pass
    tot = sum(agg.values())
    print("total samples", tot)
    for spec in ranges:
        loc, name = spec.split("=")
        fn, span = loc.split(":")
        a, b = (int(x) for x in span.split("-"))
        v = sum(c for (ff, ln), c in agg.items() if ff == fn and a <= ln <= b)
        print(f"  {name:30s} {v:6d} {100 * v / max(tot, 1):5.1f}%")
    for k, v in agg.most_common(top):
        print(f"{v:6d} {100 * v / max(tot, 1):5.1f}% {k[0]}:{k[1]} {src[k].strip()[:90]}")


if __name__ == "__main__":
    main()
