"""Summarise an ncu --csv launch list (gpu__time_duration.sum, optionally dram__bytes_read/write.sum) by kernel.

    python tools/launch_summary.py launches.csv[.gz] [--last N]     # --last: only the last N launches (steady state)
"""
import collections
import csv
import gzip
import re
import sys

path = sys.argv[1]
last = int(sys.argv[sys.argv.index("--last") + 1]) if "--last" in sys.argv else 0
rows = list(csv.reader(gzip.open(path, "rt") if path.endswith(".gz") else open(path)))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ii, ki, mi, vi, ui = (h.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
UNIT = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
        "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
launches = collections.OrderedDict()  # id -> [name, us, read_MB, write_MB]
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1.0)
    m = re.search(r"(k_\w+|vectorized_elementwise_kernel|\w+_kernel)", r[ki])
    name = m.group(1) if m else r[ki][:40]
    t = re.search(r"k_\w+<([^>]*)>", r[ki])
    if t:
        name += "<" + t.group(1)[:24] + ">"
    e = launches.setdefault(r[ii], [name, 0.0, 0.0, 0.0])
    if r[mi] == "gpu__time_duration.sum":
        e[1] = v
    elif r[mi] == "dram__bytes_read.sum":
        e[2] = v
    elif r[mi] == "dram__bytes_write.sum":
        e[3] = v
items = list(launches.values())
total_all = len(items)
if last:
    items = items[-last:]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for name, us, rd, wr in items:
    a = agg[name]
    a[0] += 1
    a[1] += us
    a[2] += rd
    a[3] += wr
tot = sum(a[1] for a in agg.values()) or 1.0
print(f"# launches summarised {len(items)} of {total_all}, total {tot:.1f} us (per-launch times under ncu are serialised and "
      "cold-cache)")
print(f"{'kernel':44s} {'launches':>8s} {'mean_us':>9s} {'share':>6s} {'dram_read_MB':>13s} {'dram_write_MB':>14s}")
for k, (c, us, rd, wr) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:44s} {c:8d} {us / c:9.2f} {us / tot:6.3f} {rd / c:13.1f} {wr / c:14.1f}")
