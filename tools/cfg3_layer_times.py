"""Per-layer SVD-stage time of cfg3 (one circuit) under two tunable sets: which layers a rule helps.
python tools/cfg3_layer_times.py "jac_cluster=0" "jac_cluster=2"  -> layer, items, bound, ms_a, ms_b"""
import sys, torch, numpy as np
sys.path.insert(0, '.')
from paper_1807_07914_b200 import MpsBatch, TruncationPolicy, compile_batch, _native
from paper_1807_07914_b200.engine import SvdTimer
from paper_1807_07914_b200 import workloads as W

import os
w = W.CONFIGS[os.environ.get("CFG", "cfg3")]()
plan = compile_batch(w.programs, w.n)
specs = sys.argv[1:3] or ["jac_cluster=0", "jac_cluster=2"]
res, meta = [], []
for si, spec in enumerate(specs):
    _native._overrides.clear()
    for kv in filter(None, spec.split(",")):
        k, v = kv.split("="); _native._overrides[k] = float(v)
    best = None
    for rep in range(2):
        b = MpsBatch(1, w.n, TruncationPolicy(w.cutoff, w.max_bond))
        t = SvdTimer(512); t.attach(b)
        calls = []
        orig = b._apply_2q_layer
        def spy(its, *a, _o=orig, _c=calls, _b=b, **k):
            ub = _b.dim_ub; s, q = its[:, 0], its[:, 1]
            _c.append((len(its), int(max(ub[s, q].max(), ub[s, q + 2].max()))))
            return _o(its, *a, **k)
        b._apply_2q_layer = spy
        b.execute(plan); torch.cuda.synchronize()
        n = t.used.value
        ms = np.array([t.events[2 * i].elapsed_time(t.events[2 * i + 1]) for i in range(n)])
        best = ms if best is None else np.minimum(best, ms)
        meta = calls
    res.append(best)
print("layer items bound  vis_round  " + "  ".join(specs))
for i, (m, a, c) in enumerate(zip(meta, res[0], res[1])):
    cmax = 2 * m[1]; nb = (cmax + 15) // 16; nb += nb & 1
    print(f"{i:3d} {m[0]:4d} {m[1]:5d} {m[0] * (nb // 2):6d}   {a:8.3f} {c:8.3f}  {'<' if c < 0.97 * a else '>' if c > 1.03 * a else '='}")
print("total", res[0].sum(), res[1].sum())
