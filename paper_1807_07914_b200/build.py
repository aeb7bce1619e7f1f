"""Build ``libbmps.so`` in-tree for sm_100a (``python -m paper_1807_07914_b200.build``)."""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
SOURCES = [PKG / "csrc" / "bmps.cu", PKG / "csrc" / "bmps_plan.cpp"]
DEPS = SOURCES + sorted((PKG / "csrc").glob("*.cuh")) + [ROOT / "include" / "bmps.h", PKG / "csrc" / "libbmps.map"]
OUT = PKG / "libbmps.so"

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-shared", "-Xcompiler", "-fPIC",
    "-Xptxas", "-v",
    # export only the bmps_* C ABI (the statically linked cudart stays internal)
    "-Xlinker", "--version-script=" + str(Path(__file__).resolve().parent / "csrc" / "libbmps.map"),
]


def nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(cand).exists():
        raise RuntimeError("nvcc not found; CUDA 12.9 toolkit required")
    return cand


def up_to_date() -> bool:
    if not OUT.exists():
        return False
    t = OUT.stat().st_mtime
    return all(p.stat().st_mtime <= t for p in DEPS)


def build(force: bool = False, verbose: bool = False, out: Path | None = None,
          defines: tuple = ()) -> Path:
    """Compile libbmps.so (``out`` + ``defines``: development variants for A/B runs,
    e.g. ``-D BMPS_WARP_INNER=0``; the product library is built without them)."""
    if out is None and not defines and not force and up_to_date():
        return OUT
    target = Path(out) if out is not None else OUT
    target.parent.mkdir(parents=True, exist_ok=True)
    cmd =[nvcc(), *NVCC_FLAGS, *[f"-D{d}" for d in defines], f"-I{ROOT / 'include'}", "-o",
           str(target) + ".tmp", *map(str, SOURCES)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed ({res.returncode})")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(str(target) + ".tmp", target)
    return target


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", action="store_true")
    ap.add_argument("--out", default=None)
    ap.add_argument("-D", action="append", default=[])
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.v, out=a.out, defines=tuple(a.D)))
