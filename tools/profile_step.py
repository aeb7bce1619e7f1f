"""One bench step under cudaProfilerStart/Stop (for ncu --profile-from-start off)."""
import sys, argparse, torch
sys.path.insert(0, '.')
import bench
from paper_1807_07914_b200 import MpsBatch, TruncationPolicy, compile_batch
ap = argparse.ArgumentParser(); ap.add_argument("--replicas", type=int, default=2); ap.add_argument("--steps", type=int, default=1)
a = ap.parse_args()
R = a.replicas
b = MpsBatch(R, bench.N_QUBITS, TruncationPolicy(bench.CUTOFF, bench.CHI))
b.run([bench.prefix_program(1003 + r, bench.STEADY_LAYERS) for r in range(R)])
dims = b.host_dims()
full = [{q for q in range(8, 41) if (dims[r, q:q + 3] == 256).all()} for r in range(R)]
plans = [compile_batch([bench.bulk_layer(k, r, full[r]) for r in range(R)], 50) for k in range(a.steps + 1)]
b.execute(plans[0]); torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for k in range(a.steps):
    b.execute(plans[k + 1])
e1.record(); torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
b.check_status()
print("step ms", e0.elapsed_time(e1) / a.steps)
print("updates", sum(1 for k in range(a.steps) for p in [bench.bulk_layer(k + 1, r, full[r]) for r in range(R)] for op in p if len(op.qubits) == 2))
