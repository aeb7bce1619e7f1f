"""Summarise an ncu --metrics ... --csv launch list by kernel (time share, DRAM bytes)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hi]
data = rows[hi + 1:]
ki, mi, ni, ui = (h.index(x) for x in ('Kernel Name', 'Metric Value', 'Metric Name', 'Metric Unit'))
SC = {'nsecond': 1e-6, 'ns': 1e-6, 'usecond': 1e-3, 'us': 1e-3, 'msecond': 1.0, 'ms': 1.0,
      'second': 1e3, 's': 1e3, 'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, '': 1, 'inst': 1}
agg = collections.defaultdict(lambda: collections.defaultdict(float))
cnt = collections.Counter()
for r in data:
    if len(r) <= mi or not r[mi]:
        continue
    name = r[ki].split('(')[0].replace('void ', '')[:45]
    if r[ni] == 'gpu__time_duration.sum':
        cnt[name] += 1
    agg[name][r[ni]] += float(r[mi].replace(',', '')) * SC[r[ui]]
T = 'gpu__time_duration.sum'
tot = sum(v[T] for v in agg.values())
print(f"{'kernel':45s} {'launches':>8s} {'total ms':>10s} {'share':>6s} {'DRAM GB':>8s}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][T]):
    d = (v['dram__bytes_read.sum'] + v['dram__bytes_write.sum']) / 1e9
    print(f"{k:45s} {cnt[k]:8d} {v[T]:10.2f} {v[T] / tot:6.3f} {d:8.2f}")
print(f"{'total':45s} {sum(cnt.values()):8d} {tot:10.2f}")
