"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.defaultdict(lambda: [0, 0.0])
tot = 0.0
n = 0
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", ""))
    v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1.0)
    m = re.search(r"(k_\w+|vectorized_elementwise_kernel|\w+_kernel)", r[ki])
    name = m.group(1) if m else r[ki][:40]
    t = re.search(r"k_\w+<([^>]*)>", r[ki])
    if t:
        name += "<" + t.group(1)[:24] + ">"
    agg[name][0] += 1
    agg[name][1] += v
    tot += v
    n += 1
print(f"launches {n}  total {tot:.1f} us")
for k, (c, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:48s} {c:5d} {v:10.1f} us {100 * v / tot:5.1f}%  avg {v / c:8.2f} us")
