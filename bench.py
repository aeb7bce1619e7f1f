#!/usr/bin/env python
"""Headline benchmark: MPS two-qubit updates/s at chi=256 (contract + Jacobi SVD + split).

Workload (BASELINE.json metric, config 3): the 50-qubit depth-40 random brick
circuit (chi_max 256, cutoff 1e-10). Each replica is a different cfg3 circuit
(seed 1003 + r) evolved on the GPU to layer 25 -- the steady state where every
bulk bond sits at the chi=256 cap (untimed setup). One timed STEP applies a
"bulk brick layer" to every replica: a random 1q gate on each bulk site and a
CNOT on every bulk pair (q, q+1) whose three bonds are all 256 (17/16 pairs,
alternating parity), i.e. every two-qubit update in the step is a chi=256
update (theta 512x512, keep 256). value = updates / device time.

Rules: W warm-up steps; K timed steps bracketed by barrier + synchronize; CUDA
events on the launching stream; max over ranks; inputs (R x 100 MB states +
~1 GB workspace) exceed the 126 MB L2 so no flush is needed; nvidia-smi clocks
sampled during the timed region. ``--impl reference`` times the reference
algorithm's CPU implementation (the numpy port in oracle/, in verbatim mode =
the reference's own einsum/LAPACK calls) on a bounded sample of the same step.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CHI = 256
N_QUBITS = 50
CUTOFF = 1e-10
BULK = (8, 41)          # pairs (q, q+1) with q in [8, 40]: dims[q..q+2] all 256 at steady state
STEADY_LAYERS = 25
FP64_PEAK_TFLOPS = 36.8  # measured: cuBLAS ZGEMM 4096^3 on this pool's B200 (tools/fp64_peaks.py)


def nominal_update_flops(dl: int, dm: int, dr: int, keep: int) -> float:
    """complex GEMM + gate mix + Golub-Kahan thin SVD (x4 complex)."""
    m, n = 2 * dl, 2 * dr
    p, q = min(m, n), max(m, n)
    return 32.0 * dl * dm * dr + 128.0 * dl * dr + 4.0 * (14.0 * q * p * p + 8.0 * p ** 3)


def svd_flops(dl: int, dr: int) -> float:
    """SURVEY.md §8(d) F_svd: Golub-Kahan thin SVD with U1 and V, x4 for complex."""
    m, n = 2 * dl, 2 * dr
    p, q = min(m, n), max(m, n)
    return 4.0 * (14.0 * q * p * p + 8.0 * p ** 3)


def update_bytes(dl: int, dm: int, dr: int, keep: int) -> float:
    return 16.0 * (2 * dl * dm + 2 * dm * dr + 2 * dl * keep + 2 * keep * dr) + 8.0 * (dl + dm + dr + keep)


def prefix_program(seed: int, layers: int):
    from paper_1807_07914_b200.workloads import brick_circuit
    rng = np.random.default_rng(np.random.SeedSequence(seed).spawn(4)[0])
    return brick_circuit(N_QUBITS, layers, rng)


def bulk_layer(step: int, replica: int, full=None):
    """One bulk brick layer (1q layer on bulk sites + CNOTs on all-256 bulk pairs).

    ``full`` (optional) is the set of sites q whose bonds q, q+1, q+2 are all at
    the cap for this replica; CNOTs on other pairs are dropped so every update
    in the step is a chi=256 update.
    """
    from paper_1807_07914_b200.ir import GateKind, Instruction
    from paper_1807_07914_b200.workloads import ONE_QUBIT_POOL
    rng = np.random.default_rng([7, step, replica])
    lo, hi = BULK
    prog = []
    for q in range(lo, hi + 1):
        name = ONE_QUBIT_POOL[int(rng.integers(len(ONE_QUBIT_POOL)))]
        kind = GateKind(name)
        params = (float(rng.uniform(0, 2 * np.pi)),) if kind.num_params else ()
        prog.append(Instruction(kind, (q,), params))
    start = lo + (step % 2)
    for q in range(start, hi, 2):
        if full is None or q in full:
            prog.append(Instruction(GateKind.CNOT, (q, q + 1)))
    return prog


def n_updates(prog) -> int:
    return sum(1 for op in prog if len(op.qubits) == 2)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms (B200_PROFILING.md)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._proc = None

    def __enter__(self):
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except FileNotFoundError:
            self._proc = None
        return self

    def _read(self):
        for line in self._proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.samples.append(parts)

    def __exit__(self, *exc):
        if self._proc:
            time.sleep(0.25)
            self._proc.terminate()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def cpu_baseline_sample(states, seconds_target: float = 15.0):
    """Time the reference algorithm (verbatim numpy/LAPACK calls) on chi=256 updates."""
    from oracle.mps_oracle import OracleMps, oracle_gate_matrix
    gam, lam = states
    o = OracleMps(N_QUBITS, CUTOFF, CHI, verbatim=True)
    o.gammas = [np.array(g) for g in gam]
    o.lams = [np.array(v) for v in lam]
    prog = [op for op in bulk_layer(0, 0) if len(op.qubits) == 2]
    done, t0 = 0, time.perf_counter()
    for op in prog:
        o.apply_2q(oracle_gate_matrix(op), op.qubits[0])
        done += 1
        if time.perf_counter() - t0 > seconds_target:
            break
    dt = time.perf_counter() - t0
    return done, dt


def run_reference(args) -> None:
    """--impl reference: the reference CPU algorithm on a bounded sample, rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle.mps_oracle import OracleMps, oracle_gate_matrix
    t_setup = time.perf_counter()
    o = OracleMps(N_QUBITS, CUTOFF, CHI, verbatim=False)
    o.run(prefix_program(1003, STEADY_LAYERS))   # untimed setup (fast contraction order)
    setup_s = time.perf_counter() - t_setup
    o.verbatim = True
    per_step = args.ref_updates
    times = []
    for k in range(args.warmup + args.steps):
        ops = [op for op in bulk_layer(k, 0) if len(op.qubits) == 2][:per_step]
        t0 = time.perf_counter()
        for op in ops:
            o.apply_2q(oracle_gate_matrix(op), op.qubits[0])
        if k >= args.warmup:
            times.append(time.perf_counter() - t0)
    total = sum(times)
    value = per_step * len(times) / total
    cores = os.cpu_count()
    line = {
        "impl": "reference", "metric": "MPS 2-qubit gate updates/sec at chi=256 (contract+SVD)",
        "value": value, "unit": "updates/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * total / len(times), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": {"workload": "cfg3 steady-state bulk brick layer (chi=256)", "n": N_QUBITS,
                   "chi_max": CHI, "cutoff": CUTOFF, "updates_per_step": per_step,
                   "steady_layers": STEADY_LAYERS, "setup_s": setup_s},
        "cpu_baseline": {"value": value, "unit": "updates/s", "cores": cores, "kind": "port",
                         "sample": f"{per_step} chi=256 updates per step, verbatim reference einsum+zgesdd "
                                   f"(oracle/mps_oracle.py verbatim=True), OpenBLAS threads default"},
        "e2e": {"value": value, "unit": "updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--replicas", type=int, default=16)
    ap.add_argument("--ref-updates", type=int, default=2)
    ap.add_argument("--mode", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-circuit", action="store_true")
    ap.add_argument("--param", action="append", default=[], help="libbmps tunable name=value")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_1807_07914_b200 import MpsBatch, TruncationPolicy, compile_batch, _native

    lib = _native.load()
    for kv in args.param:
        k, v = kv.split("=")
        assert lib.bmps_set_param(k.encode(), float(v)) == 0, kv
    R = args.replicas
    policy = TruncationPolicy(CUTOFF, CHI)
    batch = MpsBatch(R, N_QUBITS, policy)
    # untimed setup: each replica a different cfg3 circuit, evolved to the steady state
    seeds = [1003 + rank * R + r for r in range(R)]
    batch.run([prefix_program(s, STEADY_LAYERS) for s in seeds])
    batch.check_status()
    dims = batch.host_dims()
    lo, hi = BULK
    full = [{q for q in range(lo, hi) if (dims[r, q:q + 3] == CHI).all()} for r in range(R)]

    total_steps = args.warmup + args.steps
    layers = [[bulk_layer(k, r, full[r]) for r in range(R)] for k in range(total_steps)]
    plans = [compile_batch(layers[k], N_QUBITS) for k in range(total_steps)]
    upd = [sum(n_updates(p) for p in layers[k]) for k in range(total_steps)]
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for k in range(args.warmup):
        batch.execute(plans[k], mode=args.mode)
    batch.check_status()
    barrier()
    # live device time of the dominant stage (K3, the SVD) from CUDA events the
    # library records on its launch stream around that stage of every update batch
    svd_ms, svd_n = ctypes.c_double(0.0), ctypes.c_int32(0)
    lib.bmps_svd_time(ctypes.byref(svd_ms), ctypes.byref(svd_n))
    lib.bmps_set_param(b"time_svd", 1.0)
    l0 = lib.bmps_launch_count()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for k in range(args.warmup, total_steps):
            batch.execute(plans[k], mode=args.mode)
        e1.record(stream)
        barrier()
    launches = int(lib.bmps_launch_count() - l0)
    lib.bmps_set_param(b"time_svd", 0.0)
    lib.bmps_svd_time(ctypes.byref(svd_ms), ctypes.byref(svd_n))
    svd_launch_ms = svd_ms.value / max(svd_n.value, 1)
    ms = e0.elapsed_time(e1)
    batch.check_status()
    sw = batch.last_sweeps(int(upd[total_steps - 1]))
    n_upd = sum(upd[args.warmup:])
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot = torch.tensor([float(n_upd)], dtype=torch.float64, device="cuda")
        dist.all_reduce(tot)
        n_upd_all = float(tot.item())
    else:
        n_upd_all = float(n_upd)
    ms_max = float(t.item())
    value = n_upd_all / (ms_max / 1e3)

    # e2e: through the public API from host program lists, H2D of the plan + D2H of results
    import torch as _t
    e2e_steps = [bulk_layer(args.warmup + k, r, full[r]) for k in range(args.steps) for r in range(R)]
    lam_host = _t.empty(batch.lam.shape, dtype=batch.lam.dtype, pin_memory=True)
    err_host = _t.empty(batch.trunc_err.shape, dtype=batch.trunc_err.dtype, pin_memory=True)
    h2d = d2h = 0
    barrier()
    t_w0 = time.perf_counter()
    f0 = _t.cuda.Event(enable_timing=True)
    f1 = _t.cuda.Event(enable_timing=True)
    f0.record(stream)
    for k in range(args.steps):
        progs = e2e_steps[k * R:(k + 1) * R]
        plan = compile_batch(progs, N_QUBITS)
        h2d = sum(a.nbytes for a in (plan.items1, plan.gates1, plan.items2, plan.gates2, plan.logidx2, plan.ranges))
        batch.execute(plan, mode=args.mode)
        lam_host.copy_(batch.lam, non_blocking=True)
        err_host.copy_(batch.trunc_err, non_blocking=True)
        d2h = lam_host.numel() * 8 + err_host.numel() * 8
    f1.record(stream)
    barrier()
    e2e_ms = max(f0.elapsed_time(f1), 1e3 * (time.perf_counter() - t_w0))
    # whole job like `value`: updates of all ranks over the slowest rank's time
    e2e_t = torch.tensor([e2e_ms, float(sum(n_updates(p) for p in e2e_steps))], dtype=torch.float64,
                         device="cuda")
    if world > 1:
        e2e_max = e2e_t[:1].clone()
        dist.all_reduce(e2e_max, op=dist.ReduceOp.MAX)
        dist.all_reduce(e2e_t)
        e2e_t[0] = e2e_max[0]
    e2e_value = float(e2e_t[1].item()) / (float(e2e_t[0].item()) / 1e3)

    # BASELINE config 4's circuits/s, sharded by circuit: a 256 x N-circuit
    # job, circuits dealt round-robin to the N ranks (weak scaling), the public batched
    # path incl. host planning: simulate_batch + <Z0 Z31> + 16 amplitudes per circuit and
    # one D2H of the results; wall clock between barriers (= the slowest rank)
    cfg4 = None
    if not args.no_circuit:
        from paper_1807_07914_b200 import workloads as W
        from paper_1807_07914_b200 import simulate_batch
        per_rank = 256
        n4 = per_rank * world
        mine = list(range(rank, n4, world))
        w4 = W.config4(circuits=n4, indices=mine)
        barrier()
        t4 = time.perf_counter()
        b4 = simulate_batch(w4.programs, w4.n, TruncationPolicy(w4.cutoff, w4.max_bond))
        zz = b4.expectations(np.arange(len(mine), dtype=np.int32), w4.paulis * len(mine))
        am = b4.amplitudes(np.repeat(np.arange(len(mine), dtype=np.int32), 16),
                           [x for bs in w4.bitstrings for x in bs])
        barrier()
        dt4 = time.perf_counter() - t4
        cfg4 = {"circuits": n4, "s": dt4, "circuits_per_s": n4 / dt4, "scaling": "weak",
                "circuits_per_gpu": per_rank,
                "path": "simulate_batch (host planning included) + expectations + amplitudes, "
                        "wall clock between barriers",
                "outputs": int(zz.size + am.size) * world}
        del b4

    line = None
    if rank == 0:
        f_upd = nominal_update_flops(CHI, CHI, CHI, CHI)
        f_svd = svd_flops(CHI, CHI)
        step_achieved = f_upd * value / world / 1e12   # per GPU, whole update
        upd_per_launch = n_upd / max(svd_n.value, 1)
        achieved = f_svd * upd_per_launch / (svd_launch_ms / 1e3) / 1e12
        prof = {}
        tp = ROOT / "profiles" / "r01_traffic.json"
        if tp.exists():
            prof = json.loads(tp.read_text())
        line = {
            "metric": "MPS 2-qubit gate updates/sec at chi=256 (contract+SVD)",
            "value": value, "unit": "updates/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
            "config": {"workload": "cfg3 steady-state bulk brick layer (chi=256)", "n": N_QUBITS,
                       "depth_prefix": STEADY_LAYERS, "chi_max": CHI, "cutoff": CUTOFF,
                       "replicas_per_gpu": R, "updates_per_step_per_gpu": n_upd / args.steps,
                       "chi256_pairs_per_replica": [len(f) for f in full],
                       "l2": "inputs larger than L2 (states + workspace > 126 MB), no flush",
                       "parallelism": f"dp{world} (independent replicas)"},
            "roofline": {"bound": "tensor",
                         "kernel": "K3 SVD stage (column sort + double Householder QR + block Jacobi "
                                   "+ Q1 epilogue), one launch sequence per bulk layer",
                         "achieved": achieved, "peak": FP64_PEAK_TFLOPS,
                         "unit": "TFLOP/s", "frac": achieved / FP64_PEAK_TFLOPS,
                         "traffic": (prof["svd_dram_bytes_per_update"] * upd_per_launch
                                     if "svd_dram_bytes_per_update" in prof else None),
                         "traffic_unit": "DRAM bytes per K3 launch sequence (ncu launch list, "
                                         "profiles/r01_traffic.json, per update x updates per launch)",
                         "algorithmic_flops_per_launch": f_svd * upd_per_launch,
                         "svd_launch_ms": svd_launch_ms, "svd_share_of_step": svd_ms.value / ms,
                         "basis": f"F_svd = 4(14 q p^2 + 8 p^3) = {f_svd:.4g} flop per chi=256 update "
                                  "(SURVEY §8(d), Golub-Kahan count, not Jacobi's executed work) x "
                                  "updates per launch / live CUDA-event time of the stage; peak = "
                                  "measured FP64 (cuBLAS ZGEMM 4096^3 / DMMA probe, tools/fp64_peaks.py; "
                                  "MEASURED_PEAKS.json has no FP64 entry)",
                         "executed_fp64_tensor_flops_per_update": prof.get("fp64_tensor_flops_per_update"),
                         "step": {"achieved": step_achieved, "frac": step_achieved / FP64_PEAK_TFLOPS,
                                  "basis": f"whole update F = {f_upd:.4g} flop x updates / step time"},
                         "nominal_bytes_per_update": update_bytes(CHI, CHI, CHI, CHI)},
            "e2e": {"value": e2e_value, "unit": "updates/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h),
                    "path": "MpsBatch.execute(compile_batch(host programs)) + D2H of all bond vectors"},
            "gpu_launches": launches,
            "jacobi_sweeps_last_step": {"mean": float(sw.mean()), "max": int(sw.max()),
                                        "p50": float(np.median(sw))},
            "clocks": clk.summary(),
        }
        if world == 1:
            # SURVEY §8(d)(i) second batch size: one brick layer of ONE circuit (B ~ 24-33)
            k0 = total_steps
            single = [[bulk_layer(k0 + k, 0, full[0])] + [[] for _ in range(R - 1)] for k in range(4)]
            sp = [compile_batch(s, N_QUBITS) for s in single]
            batch.execute(sp[0], mode=args.mode)
            torch.cuda.synchronize()
            h0 = torch.cuda.Event(enable_timing=True)
            h1 = torch.cuda.Event(enable_timing=True)
            h0.record(stream)
            for p in sp[1:]:
                batch.execute(p, mode=args.mode)
            h1.record(stream)
            torch.cuda.synchronize()
            batch.check_status()
            nb = sum(n_updates(s[0]) for s in single[1:])
            line["single_circuit_layer"] = {
                "updates_per_layer": nb / 3, "updates_per_s": nb / (h0.elapsed_time(h1) / 1e3),
                "ms_per_layer": h0.elapsed_time(h1) / 3}
        if not args.no_circuit and world == 1:
            from paper_1807_07914_b200 import workloads as W
            w3 = W.config3()
            b3 = MpsBatch(1, w3.n, TruncationPolicy(w3.cutoff, w3.max_bond))
            p3 = compile_batch(w3.programs, w3.n)
            torch.cuda.synchronize()
            g0 = torch.cuda.Event(enable_timing=True)
            g1 = torch.cuda.Event(enable_timing=True)
            g0.record(stream)
            b3.execute(p3)
            g1.record(stream)
            torch.cuda.synchronize()
            line["cfg3_full_circuit"] = {"s": g0.elapsed_time(g1) / 1e3,
                                         "circuits_per_s": 1e3 / g0.elapsed_time(g1)}
            del b3
        if cfg4 is not None:
            line["cfg4_circuits"] = cfg4
        if not args.no_cpu_baseline and world == 1:
            gam = batch.site_tensors(0)
            lam = batch.bond_vectors(0)
            done, dt = cpu_baseline_sample((gam, lam))
            line["cpu_baseline"] = {"value": done / dt, "unit": "updates/s", "cores": os.cpu_count(),
                                    "kind": "port",
                                    "sample": f"{done} chi=256 updates (verbatim reference einsum + "
                                              f"zgesdd via oracle/mps_oracle.py) in {dt:.1f} s on the "
                                              "GPU box host, from replica 0's steady state"}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
