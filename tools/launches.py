"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hi]
ki, vi, ui = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
agg = collections.defaultdict(list)
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].replace('void ', '').replace('sdqz::', '').replace('<unnamed>::', '').replace('unnamed>::', '').split('(')[0]
    v = float(r[vi].replace(',', ''))
    scale = {'ns': 1e-3, 'nsecond': 1e-3, 'us': 1, 'usecond': 1, 'ms': 1e3, 'msecond': 1e3}[r[ui]]
    agg[name].append(v * scale)
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{k[:60]:60s} n={len(v):3d} avg={sum(v)/len(v):10.2f} us  share={sum(v)/tot*100:5.1f}%")
