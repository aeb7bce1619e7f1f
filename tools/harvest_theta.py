"""Harvest two-site theta matrices of a cfg3 steady state through the CPU oracle
(input of tools/jacobi_model.py): python tools/harvest_theta.py OUTDIR [LAYER] [COUNT]."""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle import mps_oracle as O
from paper_1807_07914_b200 import workloads as W

out = Path(sys.argv[1]); out.mkdir(parents=True, exist_ok=True)
layer = int(sys.argv[2]) if len(sys.argv) > 2 else 25
count = int(sys.argv[3]) if len(sys.argv) > 3 else 4
w = W.config3()
n = w.n
per_layer = lambda d: n + len(range(d % 2, n - 1, 2))
start = sum(per_layer(d) for d in range(layer))
prog = w.programs[0][: start + per_layer(layer)]
st = O.OracleMps(n, w.cutoff, w.max_bond)
saved = []
orig_svd = np.linalg.svd
def svd_hook(mat, *a, **k):
    if svd_hook.on and mat.shape == (512, 512) and len(saved) < count:
        np.save(out / f"M_{len(saved)}.npy", mat)
        saved.append(1)
    return orig_svd(mat, *a, **k)
svd_hook.on = False
np.linalg.svd = svd_hook
st.run(prog[:start])
svd_hook.on = True
st.run(prog[start:])
print("saved", len(saved), "matrices to", out, "dims", st.dims())
