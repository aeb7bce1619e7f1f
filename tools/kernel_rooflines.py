"""Roofline fractions of the hot path's secondary kernels on the bench's steady state.

The bench line's roofline object covers the dominant stage (K3, the SVD). This tool
measures the other hot-path kernels on the same input -- 16 cfg3 replicas evolved to
layer 25 (every bulk bond at chi = 256; states 16 x 100 MB, far above L2) -- each
timed with CUDA events on the launching stream over repeated launches after warm-up:

* K1 ``bmps_apply_1q`` (HBM): every (replica, site) item, 2x2 in place; algorithmic
  bytes = read + write of each site tensor at its true dims (16 B x dl x 2 x dr x 2).
* K6 ``bmps_amplitudes`` (HBM / L2): 4096 bitstrings (256 per replica); algorithmic
  bytes per bitstring = the half site tensors it contracts (16 B x dl x dr per site)
  + lambda; flops 8 dl dr per site. Bitstrings of one replica share its tensors
  through L2, so bytes/s can exceed HBM; the flop rate is the honest figure.
* K5 environment transfers (FP64 tensor, cap > 32): all identity environments of
  every replica (``MpsBatch.environments``, direction 0 and 1); flops per site
  16 dl dr (dl + dr). Timed with the host loop of launches
  inside the region (one launch pair per site), so gaps count against it.
* K2 ``theta_kernel`` / K4 ``gemm_kernel<SplitOp>``: from the committed ncu launch
  list of the bench step (``profiles/r02_step_launches.csv``), per-launch
  duration vs the nominal flops of its updates (one grid slice per chi=256 update).

Prints one JSON object; ``profiles/r01_kernel_rooflines.json`` keeps a GPU run.
Usage: python tools/kernel_rooflines.py [--launch-list CSV]
"""
from __future__ import annotations

import argparse
import csv
import json
import re
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402  (steady-state builders and constants)

HBM_FALLBACK_GBS = 7700.0


def hbm_peak() -> tuple[float, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text())["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy, burst)"
    return HBM_FALLBACK_GBS, "B200_PROFILING.md fallback"


def timed(fn, reps: int, warm: int = 3) -> float:
    import torch
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


def from_launch_list(path: Path, chi: int = 256) -> dict:
    """Per-launch theta / split rooflines from an ncu --metrics gpu__time_duration launch list."""
    rows = list(csv.reader(path.read_text().splitlines()))
    hdr = next(r for r in rows if "Kernel Name" in r)
    tot = {"theta": [0, 0.0, 0], "split": [0, 0.0, 0]}
    for r in rows:
        if len(r) != len(hdr) or r is hdr:
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"]
        key = "theta" if name.startswith("bmps::theta_kernel") else (
            "split" if "SplitOp<0>" in name else None)
        if key:
            grid = [int(x) for x in re.findall(r"\d+", d["Grid Size"])]
            items = grid[1] if key == "theta" else grid[2]   # theta (tiles, items), split (tiles, tiles, items)
            tot[key][2] += items
            tot[key][0] += 1
            tot[key][1] += float(d["Metric Value"].replace(",", "")) * (
                1e-9 if d.get("Metric Unit", "ns") in ("ns", "nsecond") else 1e-6)
    out = {}
    # theta: 2 chained complex contractions (A1 A2 then the 4x4 gate) = 32 chi^3 + 128 chi^2
    f_theta = 32.0 * chi ** 3 + 128.0 * chi ** 2
    # split: keep x (2 chi) x (2 chi) complex product (W = X0 V S^-1 or U^H X0) = 8 keep r c
    f_split = 8.0 * chi * (2 * chi) * (2 * chi)
    for key, f in (("theta", f_theta), ("split", f_split)):
        n, t, items = tot[key]
        if n == 0:
            continue
        per_launch = t / n
        # one launch per update batch; its grid holds one slice per chi=256 update
        out[key] = {"launches": n, "avg_launch_ms": per_launch * 1e3, "updates_per_launch": items / n,
                    "flops_per_launch": f * items / n,
                    "achieved_tflops": f * items / n / per_launch / 1e12}
    return out


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--launch-list", default=str(ROOT / "profiles" / "r01_step_launches_final5.csv"))
    ap.add_argument("--replicas", type=int, default=16)
    args = ap.parse_args()

    import torch
    from paper_1807_07914_b200 import MpsBatch, TruncationPolicy, _native
    from paper_1807_07914_b200.engine import _ptr, _stream

    peak_gbs, peak_src = hbm_peak()
    fp64 = bench.fp64_peak()[0]
    R, n = args.replicas, bench.N_QUBITS
    batch = MpsBatch(R, n, TruncationPolicy(bench.CUTOFF, bench.CHI))
    batch.run([bench.prefix_program(1003 + r, bench.STEADY_LAYERS) for r in range(R)])
    batch.check_status()
    dims = batch.host_dims().astype(np.int64)          # [R][n+1]
    dl, dr = dims[:, :-1], dims[:, 1:]                 # per (replica, site)
    lib = _native.load()
    res: dict = {"workload": f"{R} cfg3 replicas at layer {bench.STEADY_LAYERS} (n={n}, chi_max 256)",
                 "hbm_peak_gbs": peak_gbs, "hbm_peak_source": peak_src, "fp64_peak_tflops": fp64}

    # K1 -- every (replica, site), random unitaries
    rng = np.random.default_rng(5)
    items = np.array([(s, k) for s in range(R) for k in range(n)], dtype=np.int32)
    g = rng.normal(size=(len(items), 2, 2)) + 1j * rng.normal(size=(len(items), 2, 2))
    u = np.stack([np.linalg.qr(m)[0] for m in g]).astype(np.complex128)
    d_items = torch.from_numpy(items).cuda()
    d_gates = torch.from_numpy(u).cuda()

    def k1():
        _native.check(lib.bmps_apply_1q(_ptr(batch.gamma), _ptr(batch.dims), R, n, batch.cap,
                                        d_items.data_ptr(), d_gates.data_ptr(), len(items), _stream()),
                      "bmps_apply_1q")
    t1 = timed(k1, 20)
    b1 = float(2 * 16 * (dl * 2 * dr).sum())
    res["K1_apply1q"] = {"items": len(items), "launch_ms": t1 * 1e3, "algorithmic_bytes": b1,
                         "achieved_gbs": b1 / t1 / 1e9, "frac_hbm": b1 / t1 / 1e9 / peak_gbs,
                         "bound": "hbm"}

    # K6 -- 256 bitstrings per replica
    per = 256
    bits = rng.integers(0, 2, size=(R * per, n), dtype=np.uint8)
    sidx = torch.from_numpy(np.repeat(np.arange(R, dtype=np.int32), per)).cuda()
    dbits = torch.from_numpy(bits).cuda()
    out = torch.empty(R * per, dtype=torch.complex128, device="cuda")

    def k6():
        _native.check(lib.bmps_amplitudes(_ptr(batch.gamma), _ptr(batch.lam), _ptr(batch.dims), R, n,
                                          batch.cap, sidx.data_ptr(), dbits.data_ptr(), R * per,
                                          out.data_ptr(), _stream()), "bmps_amplitudes")
    t6 = timed(k6, 10)
    b6 = float(per * (16 * (dl * dr).sum() + 8 * dims.sum()))
    f6 = float(per * 8 * (dl * dr).sum())
    res["K6_amplitudes"] = {"bitstrings": R * per, "launch_ms": t6 * 1e3,
                            "algorithmic_bytes": b6, "achieved_gbs": b6 / t6 / 1e9,
                            "unique_bytes": float(16 * (dl * dr).sum() * 2),
                            "unique_gbs": float(16 * (dl * dr).sum() * 2) / t6 / 1e9,
                            "frac_hbm_unique": float(16 * (dl * dr).sum() * 2) / t6 / 1e9 / peak_gbs,
                            "achieved_tflops": f6 / t6 / 1e12, "bound": "hbm/L2"}

    # K5 -- identity environments of every replica, both directions
    states = np.arange(R, dtype=np.int32)
    f5 = float((16 * dl * dr * (dl + dr)).sum())
    for direction in (0, 1):
        t5 = timed(lambda: batch.environments(states, direction), 3, warm=1)
        res[f"K5_env_transfer_dir{direction}"] = {
            "sites": int(R * n), "call_ms": t5 * 1e3, "flops": f5,
            "achieved_tflops": f5 / t5 / 1e12, "frac_fp64": f5 / t5 / 1e12 / fp64,
            "bound": "tensor", "note": "host loop of per-site launches inside the timed region"}

    ll = Path(args.launch_list)
    if ll.exists():
        step = from_launch_list(ll)
        for key, v in step.items():
            v["frac_fp64"] = v["achieved_tflops"] / fp64
            v["source"] = ll.name
            res[f"{'K2_theta' if key == 'theta' else 'K4_split'}"] = v
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
