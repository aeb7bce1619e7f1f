"""Per-kernel totals of time, DRAM bytes and FP64 tensor ops from an ncu --csv launch list."""
import csv, collections, json, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hi]; data = rows[hi + 1:]
ki, mn, mv, mu, idi = (h.index(x) for x in ('Kernel Name', 'Metric Name', 'Metric Value', 'Metric Unit', 'ID'))
scale = {'ns': 1e-9, 'nsecond': 1e-9, 'us': 1e-6, 'usecond': 1e-6, 'ms': 1e-3, 'msecond': 1e-3, 's': 1.0,
         'second': 1.0, 'byte': 1, 'Kbyte': 1e3, 'KB': 1e3, 'Mbyte': 1e6, 'MB': 1e6, 'Gbyte': 1e9, 'GB': 1e9, '': 1}
per = collections.defaultdict(dict); names = {}
for r in data:
    if len(r) <= mv or not r[mv]:
        continue
    per[r[idi]][r[mn]] = float(r[mv].replace(',', '')) * scale.get(r[mu], 1)
    names[r[idi]] = r[ki].split('(')[0].replace('void ', '').replace('bmps::', '')[:44]
agg = collections.defaultdict(collections.Counter)
for i, d in per.items():
    for k, v in d.items():
        agg[names[i]][k] += v
    agg[names[i]]['launches'] += 1
T = 'gpu__time_duration.sum'; F = 'sm__ops_path_tensor_src_fp64.sum'
tot = {k: sum(a[k] for a in agg.values()) for k in (T, 'dram__bytes_read.sum', 'dram__bytes_write.sum', F)}
print(f"{'kernel':44s} {'n':>5s} {'ms':>9s} {'share':>6s} {'DRAM GB':>8s} {'FP64 TF':>8s}")
for k, a in sorted(agg.items(), key=lambda x: -x[1][T]):
    dram = (a['dram__bytes_read.sum'] + a['dram__bytes_write.sum']) / 1e9
    print(f"{k:44s} {int(a['launches']):5d} {a[T]*1e3:9.2f} {a[T]/tot[T]:6.3f} {dram:8.2f} {a[F]/max(a[T],1e-12)/1e12:8.2f}")
print(json.dumps({"time_s": tot[T], "dram_bytes": tot['dram__bytes_read.sum'] + tot['dram__bytes_write.sum'],
                  "fp64_tensor_ops": tot[F]}))
