"""profiles/<round>_traffic.json from an ncu launch list of one bench step.

Usage: python tools/make_traffic.py LAUNCHES.csv UPDATES OUT.json
The launch list must carry gpu__time_duration.sum, dram__bytes_read.sum,
dram__bytes_write.sum and sm__ops_path_tensor_src_fp64.sum per kernel
(ncu --profile-from-start off ... python tools/profile_step.py --replicas 8).
"""
import collections
import csv
import json
import sys

SC = {'nsecond': 1e-6, 'ns': 1e-6, 'usecond': 1e-3, 'us': 1e-3, 'msecond': 1.0, 'ms': 1.0, 'second': 1e3, 's': 1e3, 'byte': 1, 'Kbyte': 1e3,
      'Mbyte': 1e6, 'Gbyte': 1e9, '': 1, 'inst': 1}
SVD = ('jacobi', 'qr_', 'dq_')   # K3: column sort, QR preconditioner, Jacobi, double-QR epilogue

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hi]
ki, mi, ni, ui = (h.index(x) for x in ('Kernel Name', 'Metric Value', 'Metric Name', 'Metric Unit'))
per = collections.defaultdict(lambda: collections.defaultdict(float))
for r in rows[hi + 1:]:
    if len(r) <= mi or not r[mi]:
        continue
    name = r[ki].split('(')[0].replace('void ', '')
    per[name][r[ni]] += float(r[mi].replace(',', '')) * SC.get(r[ui], 1)
upd = int(sys.argv[2])


def tot(metric, pred=lambda n: True):
    return sum(v[metric] for n, v in per.items() if pred(n))


is_svd = lambda n: any(k in n for k in SVD)
dram = lambda pred: tot('dram__bytes_read.sum', pred) + tot('dram__bytes_write.sum', pred)
out = {
    "source": f"ncu --profile-from-start off launch list of one bench step ({sys.argv[1]})",
    "updates_in_step": upd,
    "step_ms_ncu": tot('gpu__time_duration.sum'),
    "svd_ms_ncu": tot('gpu__time_duration.sum', is_svd),
    "dram_bytes_step": dram(lambda n: True),
    "dram_bytes_per_update": dram(lambda n: True) / upd,
    "svd_dram_bytes_per_update": dram(is_svd) / upd,
    "jacobi_dram_bytes_per_update": dram(lambda n: 'jacobi' in n) / upd,
    "algorithmic_bytes_per_update": 8396800,
    "fp64_tensor_flops_per_update": tot('sm__ops_path_tensor_src_fp64.sum') / upd,
    "nominal_flops_per_update": 12356419584,
    "nominal_svd_flops_per_update": 11811160064,
    "kernels": {n: {k: v for k, v in m.items()} for n, m in per.items()},
    "note": ("svd_* covers the K3 kernels (dq_colsort, qr_panel/qr_update/qr_form_y, "
             "jacobi_dynamic, dq_sort, dq_apply_q1). sm__ops_path_tensor_src_fp64 counts flops "
             "(2 per DMMA multiply-add; 1.94e12 on the Jacobi launch of "
             "profiles/r02_jacobi_full.txt = 3.79e9 DMMA.8x8x4 x 256 x 2)."),
}
json.dump(out, open(sys.argv[3], 'w'), indent=1)
print(json.dumps({k: v for k, v in out.items() if k != 'kernels'}, indent=1))
