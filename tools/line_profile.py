"""Aggregate ncu warp-stall samples per CUDA source line (ncu --print-source cuda,sass CSV)."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
kernel_filter = sys.argv[2] if len(sys.argv) > 2 else None
cur_file, cur_fn, cur_line, cur_src = None, None, None, None
agg = collections.Counter(); src_of = {}
total = 0
for r in rows:
    if not r: continue
    if r[0] == 'File Path': cur_file = r[1].split('/')[-1]; continue
    if r[0] == 'Function Name': cur_fn = r[1]; continue
    if r[0] == 'Line No': continue
    if kernel_filter and kernel_filter not in (cur_fn or ''): continue
    if r[0]:
        cur_line = int(r[0]); cur_src = r[1]
    if len(r) > 4 and r[4].isdigit():
        key = (cur_file, cur_line)
        agg[key] += int(r[4]); total += int(r[4])
        src_of[key] = cur_src
print("total samples", total)
for (f, l), v in agg.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 40):
    print(f"{v/total:6.3f} {f}:{l:<5d} {src_of[(f, l)].strip()[:90]}")
