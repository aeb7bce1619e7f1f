"""Per-warp timeline of the inner sweep's rotation / Q-update phase (timers build):
when each warp of CTA 0 starts the phase, finishes its own work and leaves the barrier."""
import ctypes, os, sys
sys.path.insert(0, '.')
os.environ['BMPS_LIB'] = os.environ.get('TIMERS_LIB', 'tools/variants/timers.so')
import numpy as np, torch
from paper_1807_07914_b200 import _native
lib = _native.load()
from paper_1807_07914_b200 import MpsBatch, TruncationPolicy, compile_batch
from paper_1807_07914_b200 import workloads as W
w = W.config4(circuits=64)
b = MpsBatch(64, w.n, TruncationPolicy(w.cutoff, w.max_bond))
b.execute(compile_batch(w.programs, w.n)); torch.cuda.synchronize()
out = (ctypes.c_uint64 * (64 * 8 * 4))()
assert lib.bmps_inner_trace(out, 64 * 8 * 4) == 0
t = np.array(out, dtype=np.int64).reshape(64, 8, 4)
for r in range(0, 24):
    base = t[r, :, 0].min()
    print(f"round-slot {r} nact {t[r,0,3]}: " + "  ".join(
        f"w{k}:{t[r,k,0]-base:5d}/{t[r,k,1]-base:5d}/{t[r,k,2]-base:5d}" for k in range(8)))
