"""One BASELINE config's evolution under cudaProfilerStart/Stop (ncu --profile-from-start off)."""
import sys
import time

import torch

sys.path.insert(0, '.')
from paper_1807_07914_b200 import MpsBatch, TruncationPolicy, compile_batch
from paper_1807_07914_b200 import workloads as W

w = W.CONFIGS[sys.argv[1]]()
plan = compile_batch(w.programs, w.n)
b = MpsBatch(len(w.programs), w.n, TruncationPolicy(w.cutoff, w.max_bond))
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
t0 = time.perf_counter()
b.execute(plan)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
b.check_status()
print(sys.argv[1], "evolve s", time.perf_counter() - t0, "max bond", int(b.host_dims().max()))
