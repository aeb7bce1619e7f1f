"""cfg2 evolution: eager execute vs CUDA-graph replay of the same plan (new angles each time)."""
import sys, time, json
import numpy as np, torch
sys.path.insert(0, '.')
from paper_1807_07914_b200 import MpsBatch, TruncationPolicy, compile_batch
from paper_1807_07914_b200 import workloads as W
from paper_1807_07914_b200.vqe import batch_energies

w = W.config2()
pol = TruncationPolicy(w.cutoff, w.max_bond)
plans = [compile_batch(W.config2(seed=s).programs, w.n) for s in (1002, 5, 6, 7)]
S = len(w.programs)

def timed(fn, reps):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for i in range(reps): fn(i)
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps

b = MpsBatch(S, w.n, pol)
def eager(i):
    b.reset(); b.execute(plans[i % 4])
eager(0)
t_eager = timed(eager, 20)
gp = b.capture(plans[0])
def graph(i):
    p = plans[i % 4]; gp.replay(p.gates1, p.gates2)
graph(0)
t_graph = timed(graph, 20)
t_q = timed(lambda i: batch_energies(b, w.paulis, w.coeffs), 5)
t0 = time.perf_counter(); compile_batch(w.programs, w.n); t_plan = time.perf_counter() - t0
print(json.dumps({"cfg2_states": S, "layers": plans[0].n_layers, "eager_execute_ms": t_eager * 1e3,
                  "graph_replay_ms": t_graph * 1e3, "energies_query_ms": t_q * 1e3,
                  "host_planning_ms": t_plan * 1e3,
                  "energies_per_s_replay_plus_query": S / (t_graph + t_q),
                  "energies_per_s_eager_plus_query": S / (t_eager + t_q)}))
