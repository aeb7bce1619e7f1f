import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_1807_07914_b200 import TruncationPolicy, simulate_batch
from paper_1807_07914_b200 import workloads as W
n_c = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
w = W.config4(circuits=n_c)
t0 = time.perf_counter()
b = simulate_batch(w.programs, w.n, TruncationPolicy(w.cutoff, w.max_bond))
b.check_status()
torch.cuda.synchronize()
print("cfg4", n_c, "ok", time.perf_counter() - t0)
