"""Summarise an ncu launch list (gpu__time_duration.sum per kernel) -> mean us per kernel and share of the step."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]
ki, vi = h.index('Kernel Name'), h.index('Metric Value')
agg = defaultdict(list)
for r in rows[hi + 1:]:
    if len(r) > vi:
        agg[r[ki].split('(')[0][:40]].append(float(r[vi].replace(',', '')))
steps = max(len(v) for v in agg.values())
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:40s} launches={len(v):4d} mean={sum(v) / len(v) / 1e3:10.1f} us  share={sum(v) / tot * 100:5.1f}%")
