"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list (developer tool)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]
ki, vi, ui = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
agg, cnt = collections.OrderedDict(), collections.Counter()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split('(')[0][:70]
    v = float(r[vi].replace(',', ''))
    v *= {'ms': 1e3, 'us': 1.0, 'ns': 1e-3, 'usecond': 1.0, 'msecond': 1e3, 'nsecond': 1e-3}.get(r[ui], 1.0)
    agg[name] = agg.get(name, 0) + v
    cnt[name] += 1
tot = sum(agg.values())
print(f"{'ms':>10} {'share':>6} {'launches':>8}  kernel")
for k, v in sorted(agg.items(), key=lambda x: -x[1]):
    print(f"{v / 1000:10.3f} {100 * v / tot:5.1f}% {cnt[k]:8d}  {k}")
print(f"{tot / 1000:10.3f} total")
