"""Debug: replay program up to op K, then dump everything around op K."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1807_07914_b200 import MpsBatch, TruncationPolicy
from paper_1807_07914_b200.workloads import random_program
from oracle.mps_oracle import OracleMps
rng = np.random.default_rng(2024)
p6 = random_program(6, 40, rng)
K = 15
b = MpsBatch(1, 6, TruncationPolicy(0.0))
b.run([p6[:K]])
o = OracleMps(6, 0.0, None).run(p6[:K])
gam0, lam0 = b.site_tensors(0), b.bond_vectors(0)
b.run([[p6[K]]])
torch.cuda.synchronize()
cap = b.cap
ws = b._ws.cpu().numpy()
def al(x): return (x + 255) & ~255
meta = ws[:64].view(np.int32)[:12]
r, c = int(meta[0]), int(meta[1])
off = al(64); osig = off; off = al(off + 8 * 2 * cap); operm = off; off = al(off + 4 * 2 * cap); off = al(off + 256)
mat = 4 * cap * cap * 16
M0 = ws[off:off + mat].view(np.complex128)[: r * c].reshape(c, r).T
X = ws[off + al(mat):off + al(mat) + mat].view(np.complex128)[: r * c].reshape(c, r).T
sig = ws[osig:osig + 8 * c].view(np.float64)
perm = ws[operm:operm + 4 * c].view(np.int32)
np.savez('gpurun_out/dbg_op.npz', M0=M0, X=X, meta=meta, sig=sig, perm=perm,
         gam0=np.array(gam0, dtype=object), lam0=np.array(lam0, dtype=object),
         ogam=np.array(o.gammas, dtype=object), olam=np.array(o.lams, dtype=object),
         gam1=np.array(b.site_tensors(0), dtype=object), lam1=np.array(b.bond_vectors(0), dtype=object), cap=cap)
print("op", p6[K], "meta", meta.tolist(), "sig", sig, "perm", perm)
