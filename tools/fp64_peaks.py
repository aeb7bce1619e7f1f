"""Measure the FP64 roofline denominators on this pool's B200 -> profiles/fp64_peak.json.

MEASURED_PEAKS.json (driver-written) has HBM and bf16 figures only; the MPS hot
path is complex128, so bench.py divides by the numbers measured here:

* cuBLAS DGEMM 8192^3 and ZGEMM 4096^3 through torch, best of 10 (burst);
* ZGEMM 4096^3 back to back for ``--seconds`` (sustained, under the power cap);
* the DMMA (mma.sync m8n8k4 f64) and DFMA issue-rate probe tools/fp64_probe.cu
  (compiled here with nvcc for sm_100a);
* nvidia-smi clocks / throttle reasons sampled during the sustained loop.

Usage (on a GPU box): python tools/fp64_peaks.py [--seconds 6] [--out profiles/fp64_peak.json]
"""

from __future__ import annotations

import argparse
import json
import re
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def burst(dtype, n: int, reps: int = 10) -> float:
    a = torch.randn(n, n, dtype=dtype, device="cuda")
    b = torch.randn(n, n, dtype=dtype, device="cuda")
    for _ in range(3):
        a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        a @ b
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    mult = 8 if dtype.is_complex else 2
    return mult * n ** 3 / best / 1e9


def sustained(n: int, seconds: float) -> float:
    a = torch.randn(n, n, dtype=torch.complex128, device="cuda")
    b = torch.randn(n, n, dtype=torch.complex128, device="cuda")
    c = torch.empty_like(a)
    torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    reps, t0 = 0, time.perf_counter()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    while time.perf_counter() - t0 < seconds:
        for _ in range(8):
            torch.matmul(a, b, out=c)
        reps += 8
        torch.cuda.synchronize()
    e1.record()
    e1.synchronize()
    return 8 * n ** 3 * reps / e0.elapsed_time(e1) / 1e9


def dmma_probe() -> dict:
    src = ROOT / "tools" / "fp64_probe.cu"
    with tempfile.TemporaryDirectory() as d:
        exe = Path(d) / "fp64_probe"
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", str(exe),
                        str(src)], check=True, capture_output=True)
        out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout
    res = {"raw": out.strip().splitlines()}
    for key, pat in (("dfma_tflops", r"DFMA: .* ([\d.]+) TFLOP/s"), ("dmma_tflops", r"DMMA: .* ([\d.]+) TFLOP/s")):
        m = re.search(pat, out)
        if m:
            res[key] = float(m.group(1))
    return res


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=6.0)
    ap.add_argument("--out", default=str(ROOT / "profiles" / "fp64_peak.json"))
    args = ap.parse_args()
    from bench import ClockSampler
    out = {"gpu": torch.cuda.get_device_name(0), "torch": torch.__version__,
           "dgemm_n": 8192, "dgemm_tflops_burst": burst(torch.float64, 8192),
           "zgemm_n": 4096, "zgemm_tflops_burst": burst(torch.complex128, 4096)}
    with ClockSampler(0) as clk:
        out["zgemm_tflops_sustained"] = sustained(4096, args.seconds)
    out["clocks"] = clk.summary()
    out.update(dmma_probe())
    out["when"] = time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())
    out["how"] = ("torch.matmul float64 8192^3 / complex128 4096^3 (8 n^3 flop), best of 10 (burst); "
                  f"complex128 4096^3 back to back for {args.seconds} s (sustained); "
                  "tools/fp64_probe.cu DFMA / DMMA m8n8k4 issue-rate kernels")
    Path(args.out).write_text(json.dumps(out, indent=1))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
