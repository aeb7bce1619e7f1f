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
PEAKS_FILE = ROOT / "profiles" / "fp64_peak.json"   # tools/fp64_peaks.py on this pool's B200
TRAFFIC_FILE = ROOT / "profiles" / "r02_traffic.json"  # tools/make_traffic.py, final-build launch list


def fp64_peak() -> tuple[float, str]:
    """The FP64 roofline denominator: the measured SUSTAINED complex128 GEMM rate
    (cuBLAS ZGEMM back to back under the power cap, tools/fp64_peaks.py) -- the
    bench's stage is timed inside a seconds-long step. MEASURED_PEAKS.json has no
    FP64 entry and B200_PROFILING.md gives no FP64 fallback."""
    if not PEAKS_FILE.exists():
        return 36.8, "round-1 cuBLAS ZGEMM 4096^3 measurement (profiles/fp64_peak.json absent)"
    d = json.loads(PEAKS_FILE.read_text())
    return float(d["zgemm_tflops_sustained"]), (
        f"{PEAKS_FILE.relative_to(ROOT)}: cuBLAS ZGEMM {d['zgemm_n']}^3 sustained "
        f"{d['zgemm_tflops_sustained']:.2f} TFLOP/s (burst {d['zgemm_tflops_burst']:.2f}, DMMA probe "
        f"{d.get('dmma_tflops', float('nan')):.2f}), clocks {d['clocks']}")


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


def records_flops(rec) -> float:
    """Sum of SURVEY §8(d)'s nominal F(dl, dm, dr) over executed update records."""
    dl, dm, dr = (rec[k].astype(np.float64) for k in ("dl", "dm", "dr"))
    m, n = 2 * dl, 2 * dr
    p, q = np.minimum(m, n), np.maximum(m, n)
    return float(np.sum(32.0 * dl * dm * dr + 128.0 * dl * dr + 4.0 * (14.0 * q * p * p + 8.0 * p ** 3)))


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


def _host_cores() -> tuple[int, int]:
    return os.cpu_count() or 1, len(os.sched_getaffinity(0))


_POOL_STATE = None


def _pool_update(i: int) -> float:
    """Pool task: one verbatim chi=256 update on this worker's forked copy of the
    steady state, OpenBLAS single-threaded; returns its wall time."""
    from threadpoolctl import threadpool_limits
    from oracle.mps_oracle import oracle_gate_matrix
    o, ops = _POOL_STATE
    op = ops[i % len(ops)]
    with threadpool_limits(1):
        t0 = time.perf_counter()
        o.apply_2q(oracle_gate_matrix(op), op.qubits[0])
        return time.perf_counter() - t0


def _oracle_steady(gam=None, lam=None):
    from oracle.mps_oracle import OracleMps
    o = OracleMps(N_QUBITS, CUTOFF, CHI, verbatim=False)
    if gam is None:
        o.run(prefix_program(1003, STEADY_LAYERS))   # fast contraction order (setup only)
    else:
        o.gammas = [np.array(g) for g in gam]
        o.lams = [np.array(v) for v in lam]
    o.verbatim = True                                # timed: the reference's own einsum + zgesdd
    return o


def cpu_reference_rates(o, rounds: int = 2) -> dict:
    """The reference CPU path (verbatim mps.py:94-136: its einsums + LAPACK zgesdd) on
    chi=256 updates of the steady state, three ways on this host: one process with
    OpenBLAS on all cores, one process single-threaded, and a fork Pool of one
    single-threaded process per usable core (independent updates -- the replicas are
    independent states). Returns updates/s of each and the best."""
    import multiprocessing as mp
    from threadpoolctl import threadpool_limits
    from oracle.mps_oracle import oracle_gate_matrix
    global _POOL_STATE
    ops = [op for op in bulk_layer(0, 0) if len(op.qubits) == 2]
    ncpu, naff = _host_cores()
    out = {}
    for label, threads in (("1_process_all_threads", None), ("1_process_1_thread", 1)):
        with threadpool_limits(threads):
            t0 = time.perf_counter()
            for op in ops[:2]:
                o.apply_2q(oracle_gate_matrix(op), op.qubits[0])
            out[label] = 2 / (time.perf_counter() - t0)
    _POOL_STATE = (o, ops)
    with mp.get_context("fork").Pool(naff) as pool:
        pool.map(_pool_update, range(naff))          # warm (page in numpy/BLAS per worker)
        t0 = time.perf_counter()
        for _ in range(rounds):
            pool.map(_pool_update, range(naff), chunksize=1)
        out[f"pool_{naff}_processes_1_thread"] = rounds * naff / (time.perf_counter() - t0)
    _POOL_STATE = None
    best = max(out, key=out.get)
    return {"rates_updates_per_s": out, "best": best, "value": out[best], "cores": naff,
            "os_cpu_count": ncpu, "sched_getaffinity": naff}


def run_reference(args) -> None:
    """--impl reference: the reference CPU algorithm on the box's host cores, rank 0
    only. One step = one chi=256 update per usable core, run by a fork Pool of
    single-threaded processes on independent copies of the steady state (the
    reference's verbatim einsum + zgesdd via oracle/mps_oracle.py)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import multiprocessing as mp
    global _POOL_STATE
    t_setup = time.perf_counter()
    o = _oracle_steady()
    setup_s = time.perf_counter() - t_setup
    ncpu, naff = _host_cores()
    _POOL_STATE = (o, [op for op in bulk_layer(0, 0) if len(op.qubits) == 2])
    times = []
    with mp.get_context("fork").Pool(naff) as pool:
        for k in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            pool.map(_pool_update, range(k * naff, (k + 1) * naff), chunksize=1)
            if k >= args.warmup:
                times.append(time.perf_counter() - t0)
    _POOL_STATE = None
    total = sum(times)
    value = naff * len(times) / total
    line = {
        "impl": "reference", "metric": "MPS 2-qubit gate updates/sec at chi=256 (contract+SVD)",
        "value": value, "unit": "updates/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * total / len(times), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": {"workload": "cfg3 steady-state bulk brick layer (chi=256)", "n": N_QUBITS,
                   "chi_max": CHI, "cutoff": CUTOFF, "updates_per_step": naff,
                   "steady_layers": STEADY_LAYERS, "setup_s": setup_s},
        "cpu_baseline": {"value": value, "unit": "updates/s", "cores": naff, "kind": "port",
                         "sample": f"{naff} chi=256 updates per step, one per usable core: fork Pool of "
                                   f"{naff} single-threaded processes (os.cpu_count {ncpu}, "
                                   f"sched_getaffinity {naff}), verbatim reference einsum + zgesdd "
                                   f"(oracle/mps_oracle.py verbatim=True)"},
        "e2e": {"value": value, "unit": "updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _timed(fn, stream):
    import torch
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    out = fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return out, max(e0.elapsed_time(e1) / 1e3, 0.0), time.perf_counter() - t0


def config_rooflines(peak: float, world: int, rank: int, stream) -> dict:
    """Whole-config FP64 fractions: the nominal F(dl, dm, dr) of every
    two-qubit update actually executed (device records, read back once) / wall / peak.
    Two-site updates only (1q gates and queries are < 2% of each config)."""
    from paper_1807_07914_b200 import MpsBatch, TruncationPolicy, compile_batch, simulate_batch
    from paper_1807_07914_b200 import workloads as W
    out = {}
    import torch
    import torch.distributed as dist
    # cfg4: BASELINE config 4 as stated -- 1024 circuits sharded by circuit across the ranks
    # (round-robin), host planning included, plus <Z0 Z31> and 16 amplitudes per circuit
    n4 = 1024
    mine = list(range(rank, n4, world))
    w4 = W.config4(circuits=n4, indices=mine)
    # untimed warm-up on another 64-circuit set: allocator growth and first-use module loads of
    # the chi<=64 kernels are not part of the job (the timed run starts from a fresh batch)
    ww = W.config4(seed=4004, circuits=64)
    simulate_batch(ww.programs, ww.n, TruncationPolicy(ww.cutoff, ww.max_bond)).check_status()
    del ww
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    b4 = simulate_batch(w4.programs, w4.n, TruncationPolicy(w4.cutoff, w4.max_bond), keep_records=True)
    zz = b4.expectations(np.arange(len(mine), dtype=np.int32), w4.paulis * len(mine))
    am = b4.amplitudes(np.repeat(np.arange(len(mine), dtype=np.int32), 16),
                       [x for bs in w4.bitstrings for x in bs])
    torch.cuda.synchronize()
    dt4 = time.perf_counter() - t4
    f4 = sum(records_flops(b4.update_records(s)) for s in range(len(mine)))
    t = torch.tensor([dt4, f4], dtype=torch.float64, device="cuda")
    if world > 1:
        tmax = t[:1].clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        dist.all_reduce(t)
        t[0] = tmax[0]
    dt4, f4 = float(t[0]), float(t[1])
    out["cfg4"] = {"circuits": n4, "s": dt4, "circuits_per_s": n4 / dt4, "scaling": "strong",
                   "nominal_tflop": f4 / 1e12, "achieved_tflops": f4 / dt4 / 1e12,
                   "frac": f4 / dt4 / 1e12 / (peak * world),
                   "path": "simulate_batch (host planning included) + expectations + amplitudes, "
                           "wall clock between barriers, max over ranks",
                   "outputs": int(zz.size + am.size)}
    del b4
    if world == 1:
        for name, cfg in (("cfg3", W.config3()), ("cfg5", W.config5())):
            b = MpsBatch(1, cfg.n, TruncationPolicy(cfg.cutoff, cfg.max_bond), keep_records=True)
            plan = compile_batch(cfg.programs, cfg.n)
            _, dev_s, wall_s = _timed(lambda: b.execute(plan), stream)
            f = records_flops(b.update_records(0))
            out[name] = {"s": wall_s, "device_s": dev_s, "updates": int(len(b.update_records(0))),
                         "nominal_tflop": f / 1e12, "achieved_tflops": f / wall_s / 1e12,
                         "frac": f / wall_s / 1e12 / peak, "path": "MpsBatch.execute (evolution)"}
            del b
        # cfg1 / cfg2 end to end through the public API (planning, evolution, queries; the
        # second of two runs each: these are 20-70 ms jobs)
        from paper_1807_07914_b200.vqe import batch_energies
        w1, w2 = W.config1(), W.config2()
        for rep in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            b1 = simulate_batch(w1.programs, w1.n, TruncationPolicy(w1.cutoff, w1.max_bond))
            b1.expectations(np.zeros(w1.n, np.int32), w1.paulis)
            b1.amplitudes(np.zeros(64, np.int32), w1.bitstrings[0])
            torch.cuda.synchronize()
            out["cfg1"] = {"s": time.perf_counter() - t0, "outputs": w1.n + 64,
                           "path": "simulate_batch + <Z_q> + 64 amplitudes"}
            t0 = time.perf_counter()
            b2 = simulate_batch(w2.programs, w2.n, TruncationPolicy(w2.cutoff, w2.max_bond))
            e2 = batch_energies(b2, w2.paulis, w2.coeffs)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            out["cfg2"] = {"s": dt, "energies_per_s": len(e2) / dt, "vectors": len(e2),
                           "terms": len(w2.paulis), "path": "simulate_batch + batch_energies"}
            del b1, b2
    return out


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--replicas", type=int, default=16)
    ap.add_argument("--mode", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-circuit", action="store_true")
    ap.add_argument("--param", action="append", default=[], help="libbmps tunable name=value")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        # NCCL's communicator-init lines (to stderr) show each rank's device and transport
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        warm = torch.ones(1, device="cuda")
        dist.all_reduce(warm)              # communicator up before any timing

    from paper_1807_07914_b200 import MpsBatch, TruncationPolicy, compile_batch, _native
    from paper_1807_07914_b200.engine import SvdTimer

    lib = _native.load()
    for kv in args.param:
        k, v = kv.split("=")
        _native._overrides[k.strip()] = float(v)
    peak, peak_basis = fp64_peak()
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
    # live device time of the dominant stage (K3, the SVD) from CUDA events the
    # library records on its launch stream around that stage of every update batch
    timer = SvdTimer(capacity=4 * args.steps + 8)
    timer.attach(batch)
    barrier()
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
    svd_total_ms, svd_n = timer.total_ms()
    batch.svd_timer = None
    svd_launch_ms = svd_total_ms / max(svd_n, 1)
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
    e2e_steps = [bulk_layer(args.warmup + k, r, full[r]) for k in range(args.steps) for r in range(R)]
    lam_host = torch.empty(batch.lam.shape, dtype=batch.lam.dtype, pin_memory=True)
    err_host = torch.empty(batch.trunc_err.shape, dtype=batch.trunc_err.dtype, pin_memory=True)
    h2d = d2h = 0
    barrier()
    t_w0 = time.perf_counter()
    f0 = torch.cuda.Event(enable_timing=True)
    f1 = torch.cuda.Event(enable_timing=True)
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

    configs = None if args.no_circuit else config_rooflines(peak, world, rank, stream)

    line = None
    if rank == 0:
        f_upd = nominal_update_flops(CHI, CHI, CHI, CHI)
        f_svd = svd_flops(CHI, CHI)
        step_achieved = f_upd * value / world / 1e12   # per GPU, whole update
        upd_per_launch = n_upd / max(svd_n, 1)
        achieved = f_svd * upd_per_launch / (svd_launch_ms / 1e3) / 1e12
        prof = json.loads(TRAFFIC_FILE.read_text()) if TRAFFIC_FILE.exists() else {}
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
                         "achieved": achieved, "peak": peak, "peak_basis": peak_basis,
                         "unit": "TFLOP/s", "frac": achieved / peak,
                         "traffic": (prof["svd_dram_bytes_per_update"] * upd_per_launch
                                     if "svd_dram_bytes_per_update" in prof else None),
                         "traffic_unit": f"DRAM bytes per K3 launch sequence (ncu, "
                                         f"{TRAFFIC_FILE.relative_to(ROOT)}: per update x updates per launch)",
                         "algorithmic_flops_per_launch": f_svd * upd_per_launch,
                         "svd_launch_ms": svd_launch_ms, "svd_share_of_step": svd_total_ms / ms,
                         "basis": f"F_svd = 4(14 q p^2 + 8 p^3) = {f_svd:.4g} flop per chi=256 update "
                                  "(SURVEY §8(d), Golub-Kahan count, not Jacobi's executed work) x "
                                  "updates per launch / live CUDA-event time of the stage",
                         "executed_fp64_tensor_flops_per_update": prof.get("fp64_tensor_flops_per_update"),
                         "step": {"achieved": step_achieved, "frac": step_achieved / peak,
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
        if configs is not None:
            line["configs"] = configs
            line["cfg4_circuits"] = configs["cfg4"]
        if not args.no_cpu_baseline and world == 1:
            t_cpu = time.perf_counter()
            cpu = cpu_reference_rates(_oracle_steady(batch.site_tensors(0), batch.bond_vectors(0)))
            line["cpu_baseline"] = {
                "value": cpu["value"], "unit": "updates/s", "cores": cpu["cores"], "kind": "port",
                "sample": (f"chi=256 updates from replica 0's steady state, verbatim reference einsum + "
                           f"zgesdd (oracle/mps_oracle.py verbatim=True) on the GPU box host "
                           f"(os.cpu_count {cpu['os_cpu_count']}, sched_getaffinity "
                           f"{cpu['sched_getaffinity']}); best of {cpu['rates_updates_per_s']} "
                           f"= {cpu['best']}; {time.perf_counter() - t_cpu:.1f} s of CPU timing"),
                "rates": cpu["rates_updates_per_s"]}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
