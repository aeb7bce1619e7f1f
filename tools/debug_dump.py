"""Debug: replay a prefix, run one op, dump the theta matrix / Jacobi meta from the workspace."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1807_07914_b200 import MpsBatch, TruncationPolicy, _native
from paper_1807_07914_b200.workloads import config1, random_program
which = sys.argv[1]
if which == "cfg1":
    w = config1(); prog, n, pol, K = w.programs[0], w.n, TruncationPolicy(0.0, 256), 231
else:
    rng = np.random.default_rng(2024); prog = random_program(10, 400, rng); n, pol, K = 10, TruncationPolicy(0.0), 94
lib = _native.load()
for tf in [4.0, 16.0, 64.0]:
    lib.bmps_set_param(b"tol_factor", tf)
    b = MpsBatch(1, n, pol)
    b.run([prog[:K]])
    b.run([[prog[K]]])
    torch.cuda.synchronize()
    cap = b.cap
    ws = b._ws.cpu().numpy()
    def al(x): return (x + 255) & ~255
    meta = ws[:64].view(np.int32)[:12]
    print(which, "tol_factor", tf, "meta", meta.tolist(), flush=True)
    if tf == 4.0:
        r, c = int(meta[0]), int(meta[1])
        off = al(64); off = al(off + 8 * 2 * cap); off = al(off + 4 * 2 * cap); off = al(off + 256)
        mat = 4 * cap * cap * 16
        M0 = ws[off:off + mat].view(np.complex128)[: r * c].reshape(c, r).T
        X = ws[off + al(mat):off + al(mat) + mat].view(np.complex128)[: r * c].reshape(c, r).T
        np.savez(f'gpurun_out/dump_{which}.npz', M0=M0, X=X, meta=meta)
