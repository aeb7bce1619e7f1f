"""Batched VQE energies on the MPS backend (analytic mode).

Restates the analytic branch of ``R:src/mpsqvm/vqe.py:87-89``:
E = sum_k c_k <P_k>, summed left to right in term order. Parameter vectors
are independent states of one ``MpsBatch``; the Pauli terms of
every vector are evaluated with shared cached environments.
"""

from __future__ import annotations

import numpy as np

from .backends import simulate_batch
from .policy import TruncationPolicy


def energies(programs, n: int, paulis, coeffs, policy: TruncationPolicy | None = None,
             *, device=None) -> np.ndarray:
    """Energy of each program's state under H = sum_k coeffs[k] * paulis[k]."""
    batch = simulate_batch(programs, n, policy, device=device)
    return batch_energies(batch, paulis, coeffs)


def batch_energies(batch, paulis, coeffs, states=None) -> np.ndarray:
    states = np.arange(batch.S) if states is None else np.asarray(states)
    nt = len(paulis)
    sidx = np.repeat(states.astype(np.int32), nt)
    vals = batch.expectations(sidx, list(paulis) * len(states)).reshape(len(states), nt)
    coeffs = [float(c) for c in coeffs]
    out = np.empty(len(states))
    for v in range(len(states)):
        acc = 0  # python sum order, as vqe.py:89
        for c, e in zip(coeffs, vals[v]):
            acc = acc + c * float(e)
        out[v] = acc
    return out
