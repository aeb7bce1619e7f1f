"""Pauli strings and weighted sums, as consumed by the expectation kernels.

Restates the on-path part of ``R:src/mpsqvm/hamiltonian.py``: the Pauli
matrices (``:15-20``), ``pauli_matrix`` (``:23-27``) and the ``terms`` layout of
``PauliHamiltonian`` (``:34-55``). The file parser and exact diagonalisation
are out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

PAULI_CODES = {"I": 0, "X": 1, "Y": 2, "Z": 3}

_PAULI = {
    "I": np.eye(2, dtype=np.complex128),
    "X": np.array([[0, 1], [1, 0]], dtype=np.complex128),
    "Y": np.array([[0, -1j], [1j, 0]], dtype=np.complex128),
    "Z": np.array([[1, 0], [0, -1]], dtype=np.complex128),
}


def pauli_matrix(label: str) -> np.ndarray:
    try:
        return _PAULI[label]
    except KeyError:
        raise ValueError(f"unknown Pauli label {label!r}") from None


def encode_pauli(pauli: str) -> np.ndarray:
    """Pauli string -> uint8 codes (I=0, X=1, Y=2, Z=3); ValueError on bad labels."""
    try:
        return np.fromiter((PAULI_CODES[c] for c in pauli), dtype=np.uint8, count=len(pauli))
    except KeyError as exc:
        raise ValueError(f"unknown Pauli label {exc.args[0]!r}") from None


_CODE_TABLE = np.full(256, 255, dtype=np.uint8)
for _c, _v in (("I", 0), ("X", 1), ("Y", 2), ("Z", 3)):
    _CODE_TABLE[ord(_c)] = _v


def encode_paulis(paulis, n: int) -> np.ndarray:
    """Many equal-length Pauli strings -> uint8 codes [count, n] in one vectorised pass
    (same codes and errors as ``encode_pauli``)."""
    paulis = list(paulis)
    for p in paulis:
        if len(p) != n:
            raise ValueError(f"Pauli string length {len(p)} != qubit count {n}")
    if not paulis:
        return np.zeros((0, n), dtype=np.uint8)
    raw = "".join(paulis).encode("utf-8", errors="replace")
    if len(raw) != n * len(paulis):           # non-ASCII label somewhere
        for p in paulis:
            encode_pauli(p)
    codes = _CODE_TABLE[np.frombuffer(raw, dtype=np.uint8)].reshape(len(paulis), n)
    if (codes == 255).any():
        bad = int(np.argmax((codes == 255).any(axis=1)))
        encode_pauli(paulis[bad])             # raises with the offending label
    return codes


@dataclass(frozen=True)
class PauliHamiltonian:
    """H = sum_k coeff_k * P_k over ``n`` qubits (validation as ``hamiltonian.py:40-51``)."""

    terms: tuple[tuple[float, str], ...]

    def __post_init__(self) -> None:
        object.__setattr__(self, "terms", tuple((float(c), str(p)) for c, p in self.terms))
        if not self.terms:
            raise ValueError("Hamiltonian needs at least one term")
        widths = {len(p) for _, p in self.terms}
        if len(widths) != 1:
            raise ValueError(f"inconsistent Pauli string lengths: {sorted(widths)}")
        for coeff, pauli in self.terms:
            if not np.isfinite(coeff):
                raise ValueError(f"non-finite coefficient {coeff}")
            encode_pauli(pauli)

    @property
    def n(self) -> int:
        return len(self.terms[0][1])
