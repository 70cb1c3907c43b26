"""Summarise an ncu report: key SOL metrics + top stall lines (SASS) + stall totals."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(det)))
h = r[0]
si, mi, vi, ui = (h.index(k) for k in ("Section Name", "Metric Name", "Metric Value", "Metric Unit"))
keys = ["Duration", "DRAM Throughput", "Executed Ipc Active", "Issue Slots Busy", "Eligible Warps", "Warp Cycles Per Issued",
        "Executed Instructions", "Registers Per", "Active Threads", "Achieved Occupancy", "L1/TEX Cache Throughput",
        "L2 Cache Throughput", "Grid Size"]
for x in r[1:]:
    if any(k in x[mi] for k in keys):
        print(f"{x[mi][:50]:50s} {x[vi]} {x[ui]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
idx = [h.index(c) for c in cols]
ai, sc, ex = h.index("Address"), h.index("Source"), h.index("Instructions Executed")
tot = collections.Counter()
lines = []
for row in rows[2:]:
    try:
        v = [int(row[i] or 0) for i in idx]
        x = int(row[ex] or 0)
    except (ValueError, IndexError):
        continue
    for c, y in zip(cols, v):
        tot[c] += y
    lines.append((sum(v), x, row[ai][-5:], row[sc][:60],
                  sorted(((c[6:], y) for c, y in zip(cols, v) if y), key=lambda t: -t[1])[:2]))
n = sum(tot.values())
print("stalls:", [(k[6:], f"{v / n:.0%}") for k, v in tot.most_common(8)])
for ln in sorted(lines, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 12]:
    print(ln)
