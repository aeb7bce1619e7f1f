"""Dense 2^n statevector oracle -- TEST INFRASTRUCTURE ONLY.

SVD-free cross-check for small registers, restating the reference's dense
simulator ``R:src/mpsqvm/dense.py:39-54`` (qubit 0 is the most significant
index; two-qubit matrices indexed ``2*s1 + s2`` with the first listed qubit
most significant, ``R:src/mpsqvm/gates.py:3-4``).
"""

from __future__ import annotations

import numpy as np

from .mps_oracle import _P, oracle_gate_matrix


def dense_run(program, n: int) -> np.ndarray:
    if n > 24:
        raise ValueError("dense oracle capped at 24 qubits")
    psi = np.zeros((2,) * n, dtype=complex)
    psi[(0,) * n] = 1.0
    for op in program:
        kind = getattr(op, "kind", None)
        if kind is not None and kind.value == "MEASURE":
            continue
        g = oracle_gate_matrix(op)
        qs = list(op.qubits)
        k = len(qs)
        gt = g.reshape((2,) * (2 * k))
        psi = np.tensordot(gt, psi, axes=(list(range(k, 2 * k)), qs))
        psi = np.moveaxis(psi, list(range(k)), qs)
    return psi.reshape(-1)


def dense_amplitude(psi: np.ndarray, bits: str) -> complex:
    return complex(psi[int(bits, 2)])


def dense_expectation(psi: np.ndarray, pauli: str) -> float:
    n = len(pauli)
    phi = psi.reshape((2,) * n)
    for q, lab in enumerate(pauli):
        if lab != "I":
            phi = np.moveaxis(np.tensordot(_P[lab], phi, axes=([1], [q])), 0, q)
    return float(np.vdot(psi, phi.reshape(-1)).real)
