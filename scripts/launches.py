"""Summarise an ncu --metrics gpu__time_duration.sum CSV: per kernel (name, grid) count, mean, min, max (us)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi, gi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Grid Size")
d = collections.defaultdict(list)
order = []
for r in rows[hdr + 1:]:
    if len(r) > vi:
        k = (r[ki][:60], r[gi])
        if k not in d:
            order.append(k)
        d[k].append(float(r[vi].replace(",", "")) / 1000)
tot = sum(sum(v) for v in d.values())
for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
    print(f"{k[0]:60s} {k[1]:>14s} n={len(v):4d} mean={sum(v)/len(v):9.1f} min={min(v):9.1f} max={max(v):9.1f} share={sum(v)/tot:6.1%}")
