"""Debug: run the smoke circuit op by op; on the first failure dump the workspace."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1807_07914_b200 import MpsBatch, TruncationPolicy, _native
from paper_1807_07914_b200.workloads import brick_circuit
rng = np.random.default_rng(7)
n = 10
prog = brick_circuit(n, 8, rng)
b = MpsBatch(1, n, TruncationPolicy(1e-10, 16))
for i, op in enumerate(prog):
    b.run([[op]])
    torch.cuda.synchronize()
    if int(b.status[0].item()):
        print("failed at op", i, op)
        meta = b._ws[:64].cpu().numpy().view(np.int32)[:12]
        print("meta", meta.tolist())
        r, c = int(meta[0]), int(meta[1])
        cap = b.cap
        ws = b._ws.cpu().numpy()
        # layout: meta 256-aligned, sig (2cap doubles), perm (2cap ints), counter 256, M0, X
        def al(x): return (x + 255) & ~255
        off = al(64); off = al(off + 8 * 2 * cap); off = al(off + 4 * 2 * cap); off = al(off + 256)
        mat = 4 * cap * cap * 16
        M0 = ws[off:off + mat].view(np.complex128)[: r * c].reshape(c, r).T
        X = ws[off + al(mat):off + al(mat) + mat].view(np.complex128)[: r * c].reshape(c, r).T
        np.savez('gpurun_out/dbg_fail.npz', M0=M0, X=X, meta=meta)
        print("M0", M0)
        print("X", X)
        print("svd", np.linalg.svd(M0, compute_uv=False))
        break
else:
    print("no failure")
