"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hi]; data = rows[hi + 1:]
ki = h.index('Kernel Name'); mi = h.index('Metric Value'); ui = h.index('Metric Unit')
agg = collections.defaultdict(lambda: [0, 0.0])
scale = {'nsecond': 1e-6, 'ns': 1e-6, 'usecond': 1e-3, 'us': 1e-3, 'msecond': 1.0, 'ms': 1.0, 'second': 1e3, 's': 1e3}
for r in data:
    if len(r) <= mi or not r[mi]:
        continue
    name = r[ki].split('(')[0].replace('void ', '')[:50]
    agg[name][0] += 1
    agg[name][1] += float(r[mi].replace(',', '')) * scale[r[ui]]
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':50s} {'launches':>8s} {'total ms':>10s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:50s} {v[0]:8d} {v[1]:10.2f} {v[1] / tot:6.3f}")
print(f"{'total':50s} {sum(v[0] for v in agg.values()):8d} {tot:10.2f}")
