"""Dynamic Jacobi phase breakdown on cfg4 (chi <= 64 circuits) from a -DBMPS_PHASE_TIMERS
build: per-visit Gram / inner / apply cycles, claims, skips, inner rounds."""
import ctypes, os, sys, time
sys.path.insert(0, '.')
os.environ['BMPS_LIB'] = os.environ.get('TIMERS_LIB', 'tools/variants/timers.so')
import torch
from paper_1807_07914_b200 import _native
lib = _native.load()
from paper_1807_07914_b200 import MpsBatch, TruncationPolicy, compile_batch
from paper_1807_07914_b200 import workloads as W
n_c = int(sys.argv[1]) if len(sys.argv) > 1 else 256
w = W.config4(circuits=n_c)
plan = compile_batch(w.programs, w.n)
b = MpsBatch(n_c, w.n, TruncationPolicy(w.cutoff, w.max_bond))
out0 = (ctypes.c_uint64 * 24)(); torch.cuda.synchronize(); lib.bmps_phase_cycles(out0)
t0 = time.perf_counter(); b.execute(plan); torch.cuda.synchronize(); dt = time.perf_counter() - t0
out1 = (ctypes.c_uint64 * 24)(); lib.bmps_phase_cycles(out1)
d = [out1[i] - out0[i] for i in range(24)]
v = max(d[3], 1); claims = max(d[11], 1); rounds = max(d[6], 1)
print(f"cfg4 {n_c} circuits evolve {dt:.3f} s; visits {d[3]} claims {d[11]} skips {d[13]}")
print(f"per visit: gram {d[0]/v:.0f} inner {d[1]/v:.0f} apply {d[2]/v:.0f}; per claim {d[10]/claims:.0f}; idle {d[12]/v:.0f} per visit")
if d[20]: print(f"phase S per round (group 0, lane 0): shuffles {d[16]/d[20]:.0f}, rotation {d[17]/d[20]:.0f}, ballot+sync {d[18]/d[20]:.0f}, updates+sync {d[19]/d[20]:.0f} cycles")
print(f"inner rounds {d[6]} ({d[6]/v:.1f} per visit): rotation+count {d[4]/rounds:.0f}, update+sync {d[5]/rounds:.0f} cycles per round")
import numpy as np
rec = b.update_records(0)
cols = np.minimum(2 * rec['dl'], 2 * rec['dr']).astype(int)
print("circuit 0 updates by Jacobi columns:", {int(c): int((cols == c).sum()) for c in sorted(set(cols.tolist()))})
