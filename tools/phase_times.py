"""Jacobi phase breakdown with the -DBMPS_PHASE_TIMERS build (tools/libbmps_timers.so)."""
import ctypes, sys, shutil, numpy as np, torch
sys.path.insert(0, '.')
from paper_1807_07914_b200 import _native
_native.LIB_PATH = __import__('pathlib').Path(__import__('os').environ.get('TIMERS_LIB', 'tools/libbmps_timers.so'))
lib = _native.load()
import bench
from paper_1807_07914_b200 import MpsBatch, TruncationPolicy, compile_batch
R = 8
b = MpsBatch(R, 50, TruncationPolicy(1e-10, 256))
b.run([bench.prefix_program(1003 + r, 25) for r in range(R)])
dims = b.host_dims()
full = [{q for q in range(8, 41) if (dims[r, q:q + 3] == 256).all()} for r in range(R)]
plan = compile_batch([bench.bulk_layer(0, r, full[r]) for r in range(R)], 50)
out0 = (ctypes.c_uint64 * 24)()
torch.cuda.synchronize(); lib.bmps_phase_cycles(out0)
b.execute(plan); torch.cuda.synchronize()
out1 = (ctypes.c_uint64 * 24)(); lib.bmps_phase_cycles(out1)
d = [out1[i] - out0[i] for i in range(8)]
tot = d[0] + d[1] + d[2]
print("visits", d[3], "cycles/visit gram %.0f inner %.0f apply %.0f" % (d[0]/d[3], d[1]/d[3], d[2]/d[3]),
      "shares gram %.2f inner %.2f apply %.2f" % (d[0]/tot, d[1]/tot, d[2]/tot))
print("inner rounds", d[6], "cycles/round: rotation+sync %.0f, update+sync %.0f (updates only in rounds with rotations)" % (d[4]/max(d[6],1), d[5]/max(d[6],1)))
