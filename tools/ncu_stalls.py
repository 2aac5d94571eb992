"""Stall-reason totals and the hottest SASS lines of one kernel in an ncu report (dev tool).

    python tools/ncu_stalls.py report.ncu-rep [min_samples]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
thr = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = [k for k, r in enumerate(rows) if r and r[0] == "Address"][0]
hdr = rows[hi]
si = hdr.index("Warp Stall Sampling (All Samples)")
ex = hdr.index("Instructions Executed")
st = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
body = [r for r in rows[hi + 1:] if len(r) > si and r[si].isdigit()]
tot = sum(int(r[si]) for r in body)
agg = {}
for r in body:
    for i in st:
        agg[hdr[i][6:]] = agg.get(hdr[i][6:], 0) + int(r[i] or 0)
print("samples", tot, "instructions", len(body))
print("stalls:", ", ".join(f"{k} {100 * v / max(tot, 1):.0f}%" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8]))
for r in body:
    v = int(r[si])
    if v < thr:
        continue
    reasons = sorted(((int(r[i] or 0), hdr[i][6:]) for i in st), reverse=True)[:3]
    print(f"{v:5d} {r[ex]:>7s} {r[1].strip()[:60]:60s} {reasons}")
