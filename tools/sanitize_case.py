"""Smallest cases that reach every hot-path kernel, for compute-sanitizer runs.

    compute-sanitizer --tool {memcheck,racecheck,synccheck,initcheck} \
        python tools/sanitize_case.py [--part all|jacobi|queries]

* ``jacobi``: a 12-qubit brick circuit at chi 64 (128-column two-site matrices:
  column sort, both Householder QRs with shared-memory and L2 panels, the
  dynamic work-claiming block Jacobi, the double-QR epilogue, finalize + split),
  the same through forced 2- and 4-CTA row-split cluster visits, and small bonds
  (<= 64 columns: the single-CTA Jacobi);
* ``queries``: K1 1q updates, K6 amplitudes, sampling, conditional_prob_zero,
  K5 expectations through both the fused sweep (cap <= 32) and the DMMA
  environment transfers (cap > 32), the dense backend.

Exit code 0 and the sanitizer's "ERROR SUMMARY: 0 errors" line are the evidence
(logs under profiles/).
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_1807_07914_b200 import (MpsBatch, TruncationPolicy, _native, dense_run,  # noqa: E402
                                   mps_run)
from paper_1807_07914_b200.workloads import brick_circuit, random_bitstrings  # noqa: E402


def jacobi_part() -> None:
    rng = np.random.default_rng(1)
    prog = brick_circuit(12, 10, rng)
    for kw in ({}, {"jac_cluster": 2}, {"jac_cluster": 4}, {"jac_cluster": 0}):
        with _native.tunables(**kw):
            st = mps_run(prog, 12, TruncationPolicy(1e-10, 64))
            st.synchronize()
            print(kw, "dims", [len(v) for v in st.bond_vectors])
    b = MpsBatch(3, 10, TruncationPolicy(1e-12, 16))
    b.run([brick_circuit(10, 6, rng) for _ in range(3)])
    b.check_status()


def queries_part() -> None:
    rng = np.random.default_rng(2)
    n = 12
    prog = brick_circuit(n, 10, rng)
    for chi in (16, 64):
        st = mps_run(prog, n, TruncationPolicy(1e-10, chi))
        st.amplitudes(random_bitstrings(n, 8, rng))
        st.expectations_pauli(["Z" + "I" * (n - 2) + "Z", "X" * n, "I" * n])
        st.expectation_pauli("Y" + "I" * (n - 1))
        st.sample(64, np.random.default_rng(3))
        st.conditional_prob_zero(np.ones(1, complex), 0)
    d = dense_run(prog[:40], n)
    d.expectation_pauli("Z" * n)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--part", default="all", choices=["all", "jacobi", "queries"])
    a = ap.parse_args()
    if a.part in ("all", "jacobi"):
        jacobi_part()
    if a.part in ("all", "queries"):
        queries_part()
    print("sanitize case done")


if __name__ == "__main__":
    main()
