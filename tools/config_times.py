"""Wall/device time of every BASELINE config end to end on one GPU (evolution + queries)."""
import json, sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_1807_07914_b200 import MpsBatch, TruncationPolicy, compile_batch, simulate_batch
from paper_1807_07914_b200 import workloads as W
from paper_1807_07914_b200.vqe import batch_energies

def timed(fn):
    torch.cuda.synchronize(); t0 = time.perf_counter(); out = fn(); torch.cuda.synchronize()
    return out, time.perf_counter() - t0

res = {}
which = sys.argv[1:] or ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"]
for name in [w for w in which for _ in range(2)]:   # second run of each config is the one kept (warm)
    w = W.CONFIGS[name]()
    pol = TruncationPolicy(w.cutoff, w.max_bond)
    S = len(w.programs)
    def evolve():
        b = simulate_batch(w.programs, w.n, pol)   # public batched path (chunked planning)
        b.check_status()
        return b
    b, t_ev = timed(evolve)
    if name == "cfg2":
        _, t_q = timed(lambda: batch_energies(b, w.paulis, w.coeffs))
        extra = {"energies_per_s": S / (t_ev + t_q)}
    elif name == "cfg4":
        def q():
            zz = b.expectations(np.arange(S, dtype=np.int32), w.paulis * S)
            amps = b.amplitudes(np.repeat(np.arange(S, dtype=np.int32), 16), [x for bs in w.bitstrings for x in bs])
            return zz, amps
        _, t_q = timed(q)
        extra = {"circuits_per_s": S / (t_ev + t_q)}
    elif name == "cfg1":
        _, t_q = timed(lambda: (b.expectations(np.zeros(w.n, np.int32), w.paulis), b.amplitudes(np.zeros(64, np.int32), w.bitstrings[0])))
        extra = {}
    else:
        _, t_q = timed(lambda: b.expectations(np.zeros(len(w.paulis), np.int32), w.paulis))
        extra = {}
    res[name] = {"evolve_s": round(t_ev, 3), "query_s": round(t_q, 3), "total_s": round(t_ev + t_q, 3), **extra}
    print(name, json.dumps(res[name]), flush=True)
    del b
    torch.cuda.empty_cache()
print(json.dumps(res))
