"""Debug: run the bench setup layer by layer, dump the first failing Jacobi item."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
import bench
from paper_1807_07914_b200 import MpsBatch, TruncationPolicy, compile_batch
from paper_1807_07914_b200.engine import asap_layers
R = 8
b = MpsBatch(R, 50, TruncationPolicy(1e-10, 256))
progs = [bench.prefix_program(1003 + r, 25) for r in range(R)]
plan = compile_batch(progs, 50)
# execute layer by layer by slicing the plan
import copy
def al(x): return (x + 255) & ~255
for L in range(plan.n_layers):
    p = copy.copy(plan)
    p.n_layers = 1
    p.off1 = np.array([plan.off1[L], plan.off1[L + 1]]) - plan.off1[L]
    p.off2 = np.array([plan.off2[L], plan.off2[L + 1]]) - plan.off2[L]
    p.items1 = plan.items1[plan.off1[L]:plan.off1[L + 1]]; p.gates1 = plan.gates1[plan.off1[L]:plan.off1[L + 1]]
    a, e = plan.off2[L], plan.off2[L + 1]
    p.items2 = plan.items2[a:e]; p.gates2 = plan.gates2[a:e]
    p.logidx2 = np.arange(e - a, dtype=np.int32); p.ranges = np.zeros((0, 3), np.int32); p.n_records = e - a
    b.execute(p)
    torch.cuda.synchronize()
    nit = e - a
    if nit == 0:
        continue
    ws = b._ws.cpu().numpy()
    meta = ws[:80 * nit].view(np.int32).reshape(nit, 20)
    bad = np.nonzero(meta[:, 7])[0]
    sweeps = meta[:, 8]
    print("layer", L, "items", nit, "max sweeps", sweeps.max(), "mean", sweeps.mean(), flush=True)
    if len(bad):
        i = int(bad[0]); cap = b.cap
        r, c = int(meta[i, 0]), int(meta[i, 1])
        off = al(80 * nit); off = al(off + 8 * 2 * cap * nit); off = al(off + 4 * 2 * cap * nit); off = al(off + 256)
        mat = 4 * cap * cap * 16
        M0 = ws[off + i * mat: off + i * mat + r * c * 16].view(np.complex128).reshape(c, r).T
        xo = al(off + mat * nit)
        X = ws[xo + i * mat: xo + i * mat + r * c * 16].view(np.complex128).reshape(c, r).T
        np.savez('gpurun_out/dump_bench.npz', M0=M0, X=X, meta=meta[i])
        print("FAIL item", i, meta[i].tolist(), "item", p.items2[i])
        break
