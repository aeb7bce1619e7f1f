"""cfg4 circuits/s through simulate_batch for several planning/launch slice sizes."""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_1807_07914_b200 import workloads as W, simulate_batch, TruncationPolicy
for S in (256, 1024):
    w4 = W.config4(circuits=S)
    for chunk in (S, S // 4, S // 8, None):
        for rep in range(2):
            torch.cuda.synchronize(); t = time.perf_counter()
            b = simulate_batch(w4.programs, w4.n, TruncationPolicy(w4.cutoff, w4.max_bond), chunk=chunk)
            zz = b.expectations(np.arange(S, dtype=np.int32), w4.paulis * S)
            torch.cuda.synchronize(); dt = time.perf_counter() - t
            b.check_status()
        print(f"S={S} chunk={chunk}: {S / dt:.1f} circuits/s ({dt:.3f} s)  <Z0Z31>[0]={float(zz[0]):.12e}", flush=True)
        del b
