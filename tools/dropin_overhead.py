"""Cost of the drop-in per-gate path (MpsState.apply_* called gate by gate, as the
reference's own callers do: R:src/mpsqvm/bench.py:99-108, tests/test_acceptance.py:61-73)
against the layered executor, on config 1 (16 qubits, 320 1q + 150 CNOT) and a
small-chi circuit; plus host vs device time of MpsBatch.execute per config."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1807_07914_b200 import MatrixGate, MpsState, TruncationPolicy, compile_batch, gate_matrix, mps_run  # noqa: E402
from paper_1807_07914_b200 import MpsBatch, workloads as W  # noqa: E402


def per_gate(prog, n, pol, planner=False):
    st = MpsState(n, pol)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for op in prog:
        g = gate_matrix(op)
        q = op.qubits
        if planner:      # round-1 path: compile_batch + pinned copies per gate
            st._batch.run([[MatrixGate(g, tuple(q))]])
        elif len(q) == 1:
            st.apply_one_qubit(g, q[0])
        else:
            st.apply_two_qubit_routed(g, q[0], q[1])
    t_host = time.perf_counter() - t0
    st.synchronize()
    return t_host, time.perf_counter() - t0


def layered(prog, n, pol):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st = mps_run(prog, n, pol)
    st.synchronize()
    return time.perf_counter() - t0


out = {}
for name, (prog, n, pol) in {
    "cfg1": (W.config1().programs[0], 16, TruncationPolicy(0.0, 256)),
    "chi16_n20": (W.brick_circuit(20, 20, np.random.default_rng(3)), 20, TruncationPolicy(1e-10, 16)),
}.items():
    per_gate(prog, n, pol)   # warm
    layered(prog, n, pol)
    h, w = per_gate(prog, n, pol)
    hp, wp = per_gate(prog, n, pol, planner=True)
    lw = layered(prog, n, pol)
    out[name] = {"gates": len(prog), "per_gate_wall_s": w, "per_gate_host_s": h,
                 "per_gate_us": 1e6 * w / len(prog), "planner_per_gate_wall_s": wp,
                 "planner_per_gate_us": 1e6 * wp / len(prog), "layered_wall_s": lw}
for name in ("cfg1", "cfg2", "cfg3", "cfg4"):
    w = W.config4(circuits=256) if name == "cfg4" else W.CONFIGS[name]()
    pol = TruncationPolicy(w.cutoff, w.max_bond)
    for rep in range(2):
        t0 = time.perf_counter()
        plan = compile_batch(w.programs, w.n)
        t1 = time.perf_counter()
        b = MpsBatch(len(w.programs), w.n, pol)
        torch.cuda.synchronize()
        l0 = b.lib.bmps_launch_count()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        t2 = time.perf_counter()
        e0.record()
        b.execute(plan)
        t3 = time.perf_counter()
        e1.record()
        torch.cuda.synchronize()
        t4 = time.perf_counter()
    out[name + "_execute"] = {"layers": plan.n_layers, "plan_ms": 1e3 * (t1 - t0),
                              "host_launch_ms": 1e3 * (t3 - t2), "device_ms": e0.elapsed_time(e1),
                              "wall_ms": 1e3 * (t4 - t2), "launches": int(b.lib.bmps_launch_count() - l0)}
print(json.dumps(out, indent=1))
