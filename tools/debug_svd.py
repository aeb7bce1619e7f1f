"""Debug: run single two-site updates on random states and dump Jacobi meta."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1807_07914_b200 import MpsBatch, TruncationPolicy, _native
from paper_1807_07914_b200.ir import MatrixGate
from paper_1807_07914_b200.workloads import haar_unitary
lib = _native.load()
tf = float(sys.argv[1]) if len(sys.argv) > 1 else 4.0
lib.bmps_set_param(b"tol_factor", tf)
rng = np.random.default_rng(0)
for dl, dm, dr in [(1, 1, 1), (1, 2, 1), (2, 2, 2), (4, 4, 4), (8, 8, 8), (16, 16, 16), (32, 32, 32), (64, 64, 64)]:
    n = 4
    b = MpsBatch(1, n, TruncationPolicy(0.0, 1024))
    g = [np.ones((1, 2, 1)), None, None, np.ones((1, 2, 1))]
    g[1] = (rng.standard_normal((dl, 2, dm)) + 1j * rng.standard_normal((dl, 2, dm)))
    g[2] = (rng.standard_normal((dm, 2, dr)) + 1j * rng.standard_normal((dm, 2, dr)))
    g[0] = (rng.standard_normal((1, 2, dl)) + 0j); g[3] = rng.standard_normal((dr, 2, 1)) + 0j
    lams = [np.sort(rng.random(dl))[::-1], np.sort(rng.random(dm))[::-1], np.sort(rng.random(dr))[::-1]]
    b.load_state(0, g, lams)
    b.run([[MatrixGate(haar_unitary(rng), (1, 2))]])
    torch.cuda.synchronize()
    meta = b._ws[:64].cpu().numpy().view(np.int32)[:12]
    print((dl, dm, dr), "meta r,c,orient,dl,dm,dr,keep,status,sweeps,conv,flag:", meta[:11].tolist(), flush=True)
