import sys, numpy as np
sys.path.insert(0, '.')
from paper_1807_07914_b200 import _native, mps_run, TruncationPolicy
from paper_1807_07914_b200.workloads import brick_circuit
w2 = int(sys.argv[1]); chi = int(sys.argv[2]); cutoff = float(sys.argv[3])
extra = {k: float(v) for k, v in (kv.split('=') for kv in sys.argv[4:])}
with _native.tunables(block_w2=w2, **extra):
    prog = brick_circuit(14, 14, np.random.default_rng(700 + chi + w2))
    st = mps_run(prog, 14, TruncationPolicy(cutoff, chi))
    st.synchronize()
    print("ok", [len(v) for v in st.bond_vectors])
