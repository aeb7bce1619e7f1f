"""Seeded synthetic workloads restating BASELINE.json ``configs``.

No public benchmark suite exists for this path; these generators produce the
circuits, parameter vectors, Hamiltonians and bitstrings of configs 1-5 from
logged seeds. Every stream comes from ``np.random.SeedSequence(seed).spawn``
so circuit, bitstring, Hamiltonian and parameter draws are independent.

The one-qubit layer follows the reference bench idiom (``R:src/mpsqvm/bench.py:52-55``):
a kind drawn uniformly from the pool, an angle U[0, 2pi) drawn only for
rotations. The brick layer of round ``d`` (0-based) uses pairs
``(a, a+1) for a in range(d % 2, n-1, 2)`` (``bench.py:56-59``) with no extra
leading H layer.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .ir import GateKind, Instruction, MatrixGate

ONE_QUBIT_POOL = ("H", "X", "Y", "Z", "RX", "RY", "RZ")


def _streams(seed: int, k: int = 4) -> list[np.random.Generator]:
    return [np.random.default_rng(s) for s in np.random.SeedSequence(seed).spawn(k)]


def haar_unitary(rng: np.random.Generator, d: int = 4) -> np.ndarray:
    """Haar-random d x d unitary: QR of a complex Gaussian with the phase fix."""
    z = (rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))) / np.sqrt(2.0)
    q, r = np.linalg.qr(z)
    diag = np.diag(r)
    return q * (diag / np.abs(diag))[np.newaxis, :]


def brick_circuit(n: int, depth: int, rng: np.random.Generator, haar_prob: float = 0.0) -> list:
    """Random 1q layer + brick nearest-neighbour layer, ``depth`` times."""
    program: list = []
    for d in range(depth):
        for q in range(n):
            name = ONE_QUBIT_POOL[int(rng.integers(len(ONE_QUBIT_POOL)))]
            kind = GateKind(name)
            params = (float(rng.uniform(0.0, 2.0 * np.pi)),) if kind.num_params else ()
            program.append(Instruction(kind, (q,), params))
        for a in range(d % 2, n - 1, 2):
            if haar_prob > 0.0 and rng.random() < haar_prob:
                program.append(MatrixGate(haar_unitary(rng), (a, a + 1)))
            else:
                program.append(Instruction(GateKind.CNOT, (a, a + 1)))
    return program


ROUND_POOL = ("X", "Y", "Z", "RX", "RY", "RZ")


def round_circuit(n: int, rounds: int, seed: int, pool: tuple = ROUND_POOL) -> list:
    """The reference's memory-scaling workload (``R:src/mpsqvm/bench.py:45-60``,
    ``generate_round_circuit``): a Hadamard layer, then per round one gate of ``pool`` on
    every qubit (angles U[0, 2 pi), drawn in the reference's order from
    ``default_rng(seed)``, so a seed names the same circuit in both code bases) and a
    CNOT brick layer starting at qubit 0 on odd rounds, at qubit 1 on even ones. Its
    acceptance laws: chi = 4 after two rounds, chi = 2^(n/2) at saturation."""
    if n < 2:
        raise ValueError("need at least 2 qubits")
    if rounds < 1:
        raise ValueError("need at least 1 round")
    rng = np.random.default_rng(seed)
    program: list = [Instruction(GateKind.H, (q,)) for q in range(n)]
    for r in range(1, rounds + 1):
        for q in range(n):
            kind = GateKind(pool[int(rng.integers(len(pool)))])
            params = (float(rng.uniform(0.0, 2.0 * np.pi)),) if kind.num_params else ()
            program.append(Instruction(kind, (q,), params))
        program += [Instruction(GateKind.CNOT, (a, a + 1)) for a in range((r + 1) % 2, n - 1, 2)]
    return program


def random_bitstrings(n: int, count: int, rng: np.random.Generator) -> list[str]:
    bits = rng.integers(0, 2, size=(count, n))
    return ["".join("1" if b else "0" for b in row) for row in bits]


@dataclass
class Workload:
    """One config instance: programs, policy and the queries to answer."""

    name: str
    n: int
    programs: list                      # list of programs (one per circuit / vector)
    cutoff: float
    max_bond: int | None
    bitstrings: list[list[str]] = field(default_factory=list)   # per program
    paulis: list[str] = field(default_factory=list)              # shared by all programs
    coeffs: np.ndarray | None = None                              # Hamiltonian coefficients
    meta: dict = field(default_factory=dict)


def config1(seed: int = 1001) -> Workload:
    """cfg1: 16 qubits, depth 20, chi_max 256, exact (cutoff 0)."""
    rc, rb, _, _ = _streams(seed)
    n = 16
    prog = brick_circuit(n, 20, rc)
    paulis = ["I" * q + "Z" + "I" * (n - q - 1) for q in range(n)]
    return Workload("cfg1", n, [prog], 0.0, 256, [random_bitstrings(n, 64, rb)], paulis,
                    meta={"seed": seed, "depth": 20})


def vqe_ansatz(theta: np.ndarray) -> list:
    """Hardware-efficient ansatz: per layer RY(theta[l, q]) on every qubit, then a CNOT ladder."""
    layers, n = theta.shape
    prog: list = []
    for layer in range(layers):
        prog.extend(Instruction(GateKind.RY, (q,), (float(theta[layer, q]),)) for q in range(n))
        prog.extend(Instruction(GateKind.CNOT, (q, q + 1)) for q in range(n - 1))
    return prog


def random_pauli_terms(n: int, count: int, rng: np.random.Generator) -> tuple[list[str], np.ndarray]:
    paulis = []
    for _ in range(count):
        w = int(rng.integers(1, 5))
        support = rng.choice(n, size=w, replace=False)
        labels = rng.integers(1, 4, size=w)
        chars = ["I"] * n
        for q, lab in zip(support, labels):
            chars[int(q)] = "XYZ"[int(lab) - 1]
        paulis.append("".join(chars))
    coeffs = rng.standard_normal(count)
    return paulis, coeffs


def config2(seed: int = 1002, batch: int = 64) -> Workload:
    """cfg2: VQE energy, 20 qubits, 4 layers, 200 Pauli terms, 64 vectors, chi_max 64, cutoff 1e-12."""
    _, _, rh, rp = _streams(seed)
    n, layers = 20, 4
    thetas = rp.uniform(-np.pi, np.pi, size=(batch, layers, n))
    paulis, coeffs = random_pauli_terms(n, 200, rh)
    progs = [vqe_ansatz(t) for t in thetas]
    return Workload("cfg2", n, progs, 1e-12, 64, [], paulis, coeffs,
                    meta={"seed": seed, "thetas": thetas})


def config3(seed: int = 1003) -> Workload:
    """cfg3: 50 qubits, depth 40, chi_max 256, cutoff 1e-10; per-site <Z>, bond profile."""
    rc, _, _, _ = _streams(seed)
    n = 50
    prog = brick_circuit(n, 40, rc)
    paulis = ["I" * q + "Z" + "I" * (n - q - 1) for q in range(n)]
    return Workload("cfg3", n, [prog], 1e-10, 256, [], paulis, meta={"seed": seed, "depth": 40})


def config4(seed: int = 1004, circuits: int = 1024, cutoff: float = 1e-4, indices=None) -> Workload:
    """cfg4: independent 32-qubit depth-24 circuits, chi_max 64, cutoff 1e-4 (reference default).

    ``indices`` builds only those circuits of the ``circuits``-circuit set (a rank's shard);
    circuit i depends on (seed, i) only.
    """
    n = 32
    children = np.random.SeedSequence(seed).spawn(circuits)
    if indices is not None:
        children = [children[i] for i in indices]
    progs, bits = [], []
    for child in children:
        rc, rb = [np.random.default_rng(s) for s in child.spawn(2)]
        progs.append(brick_circuit(n, 24, rc))
        bits.append(random_bitstrings(n, 16, rb))
    paulis = ["Z" + "I" * (n - 2) + "Z"]
    return Workload("cfg4", n, progs, cutoff, 64, bits, paulis, meta={"seed": seed})


def config5(seed: int = 1005) -> Workload:
    """cfg5: 100 qubits, depth 20, CNOT or Haar (p=1/2) per brick pair, chi_max 1024, cutoff 1e-12."""
    rc, _, _, _ = _streams(seed)
    n = 100
    prog = brick_circuit(n, 20, rc, haar_prob=0.5)
    paulis = ["I" * q + p + "I" * (n - q - 1) for p in "XZ" for q in range(n)]
    return Workload("cfg5", n, [prog], 1e-12, 1024, [], paulis, meta={"seed": seed, "depth": 20})


CONFIGS = {"cfg1": config1, "cfg2": config2, "cfg3": config3, "cfg4": config4, "cfg5": config5}


ALL_ONE_QUBIT = ("H", "X", "Y", "Z", "RX", "RY", "RZ", "I")
ALL_TWO_QUBIT = ("CNOT", "CZ", "SWAP")


def random_program(n: int, num_gates: int, rng: np.random.Generator,
                   two_qubit_prob: float = 0.4) -> list:
    """Random gate list over the full gate set, including non-adjacent pairs.

    Same distribution as the reference test fixture ``R:tests/conftest.py:20-33``
    (used for the small-n parity cases).
    """
    program: list = []
    for _ in range(num_gates):
        if n >= 2 and rng.random() < two_qubit_prob:
            kind = GateKind(ALL_TWO_QUBIT[int(rng.integers(len(ALL_TWO_QUBIT)))])
            q1, q2 = (int(q) for q in rng.choice(n, size=2, replace=False))
            program.append(Instruction(kind, (q1, q2)))
        else:
            kind = GateKind(ALL_ONE_QUBIT[int(rng.integers(len(ALL_ONE_QUBIT)))])
            params = (float(rng.uniform(0, 2 * np.pi)),) if kind.num_params else ()
            program.append(Instruction(kind, (int(rng.integers(n)),), params))
    return program
