import cProfile, pstats, sys, torch
sys.path.insert(0, '.')
from paper_1807_07914_b200 import workloads as W, MpsBatch, TruncationPolicy, compile_batch
w = W.config3(); pol = TruncationPolicy(w.cutoff, w.max_bond)
plan = compile_batch(w.programs, w.n)
b = MpsBatch(1, w.n, pol); b.execute(plan); torch.cuda.synchronize()
b = MpsBatch(1, w.n, pol); torch.cuda.synchronize()
cProfile.run("b.execute(plan)", "/tmp/ex.prof")
torch.cuda.synchronize()
pstats.Stats("/tmp/ex.prof").sort_stats("tottime").print_stats(12)
