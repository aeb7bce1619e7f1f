"""Drop-in ``MpsState`` for the reference MPS backend, backed by HBM + sm_100a kernels.

Mirrors the public surface of ``R:src/mpsqvm/mps.py:52-237`` -- constructor,
``apply_one_qubit`` / ``apply_two_qubit_adjacent`` / ``apply_two_qubit_routed``,
``amplitude``, ``expectation_pauli``, ``norm_sq``, bookkeeping and the
``site_tensors`` / ``bond_vectors`` attributes -- with the same argument
validation (``ValueError`` messages) and numerical failure reports
(``RuntimeError``). The state lives on the GPU (a one-state ``MpsBatch``);
``site_tensors`` and ``bond_vectors`` are host copies made on access.

Numerical failures detected on the device (Jacobi non-convergence, all
singular values truncated) are raised at the next host synchronisation
(any query or ``synchronize()``), not inside the asynchronous gate call.
"""

from __future__ import annotations

import numpy as np

from .engine import MpsBatch, compile_batch, lower_program
from .gates import check_unitary
from .ir import MatrixGate
from .policy import TruncationPolicy


class MpsState:
    """Vidal-form factorized wavefunction over ``n`` qubits, initially |0...0>."""

    def __init__(self, n: int, policy: TruncationPolicy | None = None, *, device=None,
                 cap: int | None = None):
        if n < 1:
            raise ValueError("need at least one qubit")
        self.n = n
        self.policy = policy or TruncationPolicy()
        self._batch = MpsBatch(1, n, self.policy, device=device, cap=cap)

    @classmethod
    def _from_batch(cls, batch: MpsBatch) -> "MpsState":
        obj = cls.__new__(cls)
        obj.n = batch.n
        obj.policy = batch.policy
        obj._batch = batch
        return obj

    # -- host views (mps.py:60-66) ---------------------------------------------
    @property
    def site_tensors(self) -> list[np.ndarray]:
        self._batch.check_status()
        return self._batch.site_tensors(0)

    @property
    def bond_vectors(self) -> list[np.ndarray]:
        self._batch.check_status()
        return self._batch.bond_vectors(0)

    @property
    def trunc_error_sq(self) -> float:
        self._batch.check_status()
        return float(self._batch.trunc_err[0].item())

    @property
    def max_bond_seen(self) -> int:
        self._batch.check_status()
        return int(self._batch.mbs[0].item())

    @property
    def peak_entries(self) -> int:
        self._batch.check_status()
        return int(self._batch.peak[0].item())

    def synchronize(self) -> None:
        """Wait for queued gates and raise any deferred numerical failure."""
        self._batch.check_status()

    # -- bookkeeping (mps.py:70-80) -----------------------------------------------
    def total_entries(self) -> int:
        d = self._batch.host_dims()[0]
        return int(sum(int(d[k]) * 2 * int(d[k + 1]) for k in range(self.n)))

    def max_bond(self) -> int:
        if self.n == 1:
            return 1
        return int(self._batch.host_dims()[0, 1:self.n].max())

    def memory_estimate_bytes(self) -> int:
        """16 bytes per complex entry, at the peak over the run so far."""
        return 16 * self.peak_entries

    # -- gate application ---------------------------------------------------------
    def _check_site(self, q: int) -> None:
        if not 0 <= q < self.n:
            raise ValueError(f"site {q} out of range for {self.n} qubits")

    def apply_one_qubit(self, gate: np.ndarray, q: int) -> None:
        """Contract a 2x2 unitary into site ``q``; bonds are untouched (mps.py:88-92)."""
        self._check_site(q)
        check_unitary(gate)
        self._batch.apply_ops(0, [(1, q, gate)])

    def apply_two_qubit_adjacent(self, gate: np.ndarray, q: int) -> None:
        """Apply a 4x4 unitary to sites ``(q, q+1)`` via contract + SVD (mps.py:94-136)."""
        self._check_site(q)
        if q + 1 >= self.n:
            raise ValueError(f"site {q} has no right neighbour (n={self.n})")
        check_unitary(gate)
        self._batch.apply_ops(0, [(2, q, gate)])

    def apply_two_qubit_routed(self, gate: np.ndarray, q1: int, q2: int) -> None:
        """Apply a 4x4 unitary to arbitrary sites, SWAP-routing if needed (mps.py:138-157)."""
        self._check_site(q1)
        self._check_site(q2)
        if q1 == q2:
            raise ValueError("two-qubit gate needs two distinct sites")
        check_unitary(gate)
        ar, site, mats = lower_program([MatrixGate(np.asarray(gate, dtype=np.complex128), (q1, q2))],
                                       self.n, validate_matrices=False)
        self._batch.apply_ops(0, list(zip(ar.tolist(), site.tolist(), mats)))

    def run(self, program) -> "MpsState":
        """Apply a whole program through the layered executor (fast path)."""
        self._batch.execute(compile_batch([program], self.n))
        return self

    # -- queries ------------------------------------------------------------------
    def amplitude(self, bits: str) -> complex:
        """<bits|psi>, with string position k addressing qubit k (mps.py:172-179)."""
        return complex(self._batch.amplitudes([0], [bits])[0])

    def amplitudes(self, bitstrings) -> np.ndarray:
        """Batched ``amplitude`` (one launch)."""
        return self._batch.amplitudes(np.zeros(len(bitstrings), np.int32), list(bitstrings))

    def norm_sq(self) -> float:
        return float(self._batch.expectations([0], ["I" * self.n])[0])

    def expectation_pauli(self, pauli: str) -> float:
        """<psi|P|psi> for a Pauli string (one of IXYZ per qubit) (mps.py:188-204)."""
        if len(pauli) != self.n:
            raise ValueError(f"Pauli string length {len(pauli)} != qubit count {self.n}")
        return float(self._batch.expectations([0], [pauli])[0])

    def expectations_pauli(self, paulis) -> np.ndarray:
        """Batched ``expectation_pauli`` with cached environments."""
        return self._batch.expectations(np.zeros(len(paulis), np.int32), list(paulis))

    def conditional_prob_zero(self, prefix_vec: np.ndarray, k: int) -> tuple[float, np.ndarray, np.ndarray]:
        """P(qubit k = 0 | fixed prefix) and the two successor prefix vectors
        (mps.py:206-214), computed on the device."""
        return self._batch.conditional_prob_zero(0, prefix_vec, k)

    def sample(self, shots: int, rng: np.random.Generator) -> dict[str, int]:
        """Full-register bitstrings by sequential conditional sampling (mps.py:216-237).

        One uniform variate is consumed per qubit per shot, in qubit order, so a
        seeded generator reproduces the reference's counts.
        """
        return self._batch.sample(0, shots, rng)
