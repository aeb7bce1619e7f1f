"""Stress the lock-free Jacobi visit scheduling under a -DBMPS_DEBUG_CHECKS build
(BMPS_LIB=tools/variants/debugchecks.so): repeated cfg4 slices (thousands of small items
per launch) and chi = 256 bench steps; a violated invariant prints BMPS_CHECK and traps."""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import bench
from paper_1807_07914_b200 import MpsBatch, TruncationPolicy, compile_batch
from paper_1807_07914_b200 import workloads as W
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
w = W.config4(circuits=256)
plan = compile_batch(w.programs, w.n)
for k in range(reps):
    b = MpsBatch(256, w.n, TruncationPolicy(w.cutoff, w.max_bond))
    b.execute(plan); b.check_status()
    del b
print("cfg4 x", reps, "ok", flush=True)
if len(sys.argv) > 2: sys.exit(0)
R = 16
b = MpsBatch(R, bench.N_QUBITS, TruncationPolicy(bench.CUTOFF, bench.CHI))
b.run([bench.prefix_program(1003 + r, bench.STEADY_LAYERS) for r in range(R)])
dims = b.host_dims()
full = [{q for q in range(8, 41) if (dims[r, q:q + 3] == 256).all()} for r in range(R)]
for k in range(reps):
    b.execute(compile_batch([bench.bulk_layer(k, r, full[r]) for r in range(R)], 50)); b.check_status()
print("chi256 steps x", reps, "ok", flush=True)
