"""Debug: run programs op by op on GPU and oracle; report the first divergence."""
import sys, itertools, numpy as np, torch
sys.path.insert(0, '.')
from paper_1807_07914_b200 import MpsBatch, TruncationPolicy
from paper_1807_07914_b200.workloads import random_program, config1
from oracle.mps_oracle import OracleMps, oracle_gate_matrix

def statevec(gam, lam):
    n = len(gam)
    v = np.ones((1, 1), complex)
    for k in range(n):
        t = gam[k] if k == n - 1 else gam[k] * lam[k][None, None, :]
        v = np.einsum('ab,bsr->asr', v, t).reshape(-1, t.shape[2])
    return v.reshape(-1)

def run_case(name, prog, n, pol):
    b = MpsBatch(1, n, pol)
    o = OracleMps(n, pol.cutoff, pol.max_bond)
    for i, op in enumerate(prog):
        o.run([op])
        b.run([[op]])
        torch.cuda.synchronize()
        st = int(b.status[0].item())
        gam, lam = b.site_tensors(0), b.bond_vectors(0)
        dims_ok = [len(x) for x in lam] == o.dims()
        if st or not dims_ok:
            print(name, "op", i, op, "status", st, "dims", [len(x) for x in lam], "ref", o.dims())
            return i, b
        if n <= 12:
            a = statevec(gam, lam); r = statevec(o.gammas, o.lams)
            err = np.max(np.abs(a - r))
            if err > 1e-9:
                print(name, "op", i, op, "statevector err", err, "norm gpu", np.vdot(a, a).real, "ref", np.vdot(r, r).real)
                print("   lam gpu", [np.round(x, 4).tolist() for x in lam])
                print("   lam ref", [np.round(x, 4).tolist() for x in o.lams])
                return i, b
    print(name, "no divergence")
    return None, b

rng = np.random.default_rng(2024)
prog = random_program(5, 20, rng)   # bonds_untouched case draws first
rng = np.random.default_rng(2024)
p6 = random_program(6, 40, rng)
run_case("norm6", p6, 6, TruncationPolicy(0.0))
rng = np.random.default_rng(2024)
p10 = random_program(10, 400, rng)
run_case("n10", p10, 10, TruncationPolicy(0.0))
w = config1()
i, b = run_case("cfg1", w.programs[0], w.n, TruncationPolicy(0.0, 256))
if i is not None:
    meta = b._ws[:64].cpu().numpy().view(np.int32)[:12]
    print("meta", meta.tolist())
