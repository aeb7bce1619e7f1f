"""Dynamic (default) Jacobi phase breakdown incl. claim / idle (-DBMPS_PHASE_TIMERS build)."""
import ctypes, sys, os, pathlib, torch
sys.path.insert(0, '.')
from paper_1807_07914_b200 import _native
os.environ['BMPS_LIB'] = os.environ.get('TIMERS_LIB', 'tools/variants/timers.so')
lib = _native.load()
import bench
from paper_1807_07914_b200 import MpsBatch, TruncationPolicy, compile_batch
R = int(sys.argv[1]) if len(sys.argv) > 1 else 16
b = MpsBatch(R, 50, TruncationPolicy(1e-10, 256))
b.run([bench.prefix_program(1003 + r, 25) for r in range(R)])
dims = b.host_dims()
full = [{q for q in range(8, 41) if (dims[r, q:q + 3] == 256).all()} for r in range(R)]
plan = compile_batch([bench.bulk_layer(0, r, full[r]) for r in range(R)], 50)
out0 = (ctypes.c_uint64 * 24)(); torch.cuda.synchronize(); lib.bmps_phase_cycles(out0)
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); b.execute(plan); e1.record(); torch.cuda.synchronize()
out1 = (ctypes.c_uint64 * 24)(); lib.bmps_phase_cycles(out1)
d = [out1[i] - out0[i] for i in range(24)]
v = max(d[3], 1); claims = max(d[11], 1)
print(f"step {e0.elapsed_time(e1):.1f} ms; visits {d[3]} claims {d[11]} skips {d[13]}")
print(f"per visit: gram {d[0]/v:.0f} inner {d[1]/v:.0f} apply {d[2]/v:.0f}; per claim: claim {d[10]/claims:.0f}; idle total {d[12]/v:.0f} per visit")
print(f"probes per claim attempt (incl. idle re-probes): {d[14] / max(d[11] + d[9], 1):.2f}; probes total {d[14]}")
rounds = max(d[6], 1)
if d[20]: print(f"phase S per round (group 0, lane 0): shuffles {d[16]/d[20]:.0f}, rotation {d[17]/d[20]:.0f}, ballot+sync {d[18]/d[20]:.0f}, updates+sync {d[19]/d[20]:.0f} cycles")
print(f"inner rounds {d[6]} ({d[6]/v:.1f} per visit): rotation+count {d[4]/rounds:.0f}, update+sync {d[5]/rounds:.0f} cycles per round")
