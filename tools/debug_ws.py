"""Debug: one small brick circuit through the dynamic Jacobi (chi up to 64 -> panels > 64 columns)."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1807_07914_b200 import MpsBatch, TruncationPolicy
from paper_1807_07914_b200.workloads import brick_circuit
n = int(sys.argv[1]) if len(sys.argv) > 1 else 12
depth = int(sys.argv[2]) if len(sys.argv) > 2 else 12
S = int(sys.argv[3]) if len(sys.argv) > 3 else 1
rng = np.random.default_rng(7)
progs = [brick_circuit(n, depth, rng) for _ in range(S)]
b = MpsBatch(S, n, TruncationPolicy(0.0, 256))
b.run(progs)
torch.cuda.synchronize()
b.check_status()
print("ok dims", b.host_dims()[0].tolist())
