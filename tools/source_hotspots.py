"""Aggregate ncu `--page source --print-source cuda,sass` CSV by CUDA source line."""
import collections
import csv
import sys

rows = list(csv.reader(sys.stdin))
hdr = None
cur_line = None
cur_src = ""
agg = collections.Counter()
src = {}
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        si = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if not hdr or len(r) < len(hdr):
        continue
    if r[0]:
        cur_line, cur_src = r[0], r[1]
    try:
        v = int(r[si] or 0)
    except ValueError:
        continue
    agg[cur_line] += v
    src[cur_line] = cur_src
tot = sum(agg.values())
print("total samples", tot)
for line, v in agg.most_common(int(sys.argv[1]) if len(sys.argv) > 1 else 20):
    print(f"{v:6d} {100 * v / max(tot, 1):5.1f}%  L{line}: {src[line].strip()[:100]}")
