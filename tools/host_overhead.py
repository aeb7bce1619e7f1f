"""Host (Python launch loop) vs device time of MpsBatch.execute for a config's evolution."""
import sys, time, torch
sys.path.insert(0, '.')
from paper_1807_07914_b200 import workloads as W, MpsBatch, TruncationPolicy, compile_batch
name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
w = W.CONFIGS[name]()
pol = TruncationPolicy(w.cutoff, w.max_bond)
for rep in range(3):
    t0 = time.perf_counter()
    plan = compile_batch(w.programs, w.n)
    t1 = time.perf_counter()
    b = MpsBatch(len(w.programs), w.n, pol)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    t2 = time.perf_counter(); e0.record()
    b.execute(plan)
    t3 = time.perf_counter(); e1.record(); torch.cuda.synchronize(); t4 = time.perf_counter()
    print(f"{name}: layers {plan.n_layers}, plan {1e3*(t1-t0):.1f} ms, execute host {1e3*(t3-t2):.1f} ms, "
          f"device {e0.elapsed_time(e1):.1f} ms, wall {1e3*(t4-t2):.1f} ms, launches/layer ~{b.lib.bmps_launch_count()}")
