"""cfg4 (batch of chi<=64 circuits) under cudaProfilerStart/Stop."""
import sys, time, torch, numpy as np
sys.path.insert(0, '.')
from paper_1807_07914_b200 import MpsBatch, TruncationPolicy, compile_batch
from paper_1807_07914_b200 import workloads as W
n_c = int(sys.argv[1]) if len(sys.argv) > 1 else 256
w = W.config4(circuits=n_c)
plan = compile_batch(w.programs, w.n)
b = MpsBatch(n_c, w.n, TruncationPolicy(w.cutoff, w.max_bond))
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
t0 = time.perf_counter()
b.execute(plan)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("cfg4", n_c, "circuits evolve s", time.perf_counter() - t0)
