"""cfg4 evolution time per libbmps tunable set: python tools/cfg4_param_sweep.py N k=v,k=v ..."""
import sys, time, torch
sys.path.insert(0, '.')
from paper_1807_07914_b200 import MpsBatch, TruncationPolicy, compile_batch, _native
from paper_1807_07914_b200 import workloads as W

n_c = int(sys.argv[1])
w = W.config4(circuits=n_c)
plan = compile_batch(w.programs, w.n)
for spec in sys.argv[2:]:
    kw = {}
    if spec != "default":
        for kv in spec.split(","):
            k, v = kv.split("=")
            kw[k] = float(v)
    _native._overrides.clear()
    _native._overrides.update(kw)
    best = None
    for rep in range(2):
        b = MpsBatch(n_c, w.n, TruncationPolicy(w.cutoff, w.max_bond))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        b.execute(plan)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        b.check_status()
        best = dt if best is None else min(best, dt)
        del b
    print(f"{spec} -> {best:.3f} s  ({n_c / best:.1f} circuits/s evolve only)", flush=True)
