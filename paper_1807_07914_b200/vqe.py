"""VQE energies and the one-parameter sweep driver on the MPS and dense backends.

Restates ``R:src/mpsqvm/vqe.py``: E = sum_k c_k <P_k> summed left to right in
term order (analytic, ``:87-89``), or with ``shots`` each non-identity term
estimated from the parity of samples of the basis-rotated state (``:40-67``,
``:90-97``) with the reference's per-term generator ``default_rng([seed, k])``.
The GPU path differs only in scheduling: every grid point (and, with shots,
every (grid point, term) state) of a ``sweep`` is one state of a shared
``MpsBatch`` (``backend="mps"``) or ``DenseBatch`` (``backend="dense"``) run in
the same launches, instead of one ``run_program`` per point. Sampling consumes the same uniforms in the same order as
``MpsState.sample`` (``mps.py:206-237``), so counts are identical.
"""

from __future__ import annotations

from dataclasses import dataclass
from math import pi, sqrt

import numpy as np

from .backends import BACKENDS, simulate_batch
from .dense import DenseBatch
from .ir import GateKind, Instruction, bind_parameters, flatten, num_qubits
from .policy import TruncationPolicy

_MAX_STATES_PER_BATCH = 4096


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
    coeffs = np.asarray([float(c) for c in coeffs], dtype=np.float64)
    if nt == 0:
        return np.zeros(len(states))
    # the reference's left-to-right Python sum (vqe.py:89): np.add.accumulate is
    # sequential, so the result is bit-identical to the scalar loop
    return np.add.accumulate(coeffs[None, :] * vals, axis=1)[:, -1].copy()


@dataclass(frozen=True)
class SweepResult:
    thetas: tuple[float, ...]
    energies: tuple[float, ...]
    argmin_theta: float
    min_energy: float


def _unitary_program(ansatz, theta: float) -> list:
    """Bound, flattened ansatz without MEASUREs (``vqe.py:30-37``)."""
    if len(ansatz.formal_params) != 1:
        raise ValueError(f"driver supports exactly one formal parameter, "
                         f"kernel '{ansatz.name}' has {len(ansatz.formal_params)}")
    program = flatten(bind_parameters(ansatz, [theta]))
    return [i for i in program if i.kind.value != "MEASURE"]


def _bound_program(ansatz, values) -> list:
    """All formal parameters of ``ansatz`` bound positionally to ``values``,
    flattened, MEASUREs dropped (``ir.py:150-184`` then ``vqe.py:37``)."""
    program = flatten(bind_parameters(ansatz, [float(v) for v in values]))
    return [i for i in program if i.kind.value != "MEASURE"]


def _basis_rotations(pauli: str) -> list[Instruction]:
    """X -> H, Y -> RZ(-pi/2) then H, Z/I -> nothing (``vqe.py:40-48``)."""
    out: list[Instruction] = []
    for q, label in enumerate(pauli):
        if label == "X":
            out.append(Instruction(GateKind.H, (q,)))
        elif label == "Y":
            out.append(Instruction(GateKind.RZ, (q,), (-pi / 2,)))
            out.append(Instruction(GateKind.H, (q,)))
    return out


def _check_backend(backend: str) -> None:
    if backend not in BACKENDS:
        raise ValueError(f"unknown backend {backend!r}; expected one of {BACKENDS}")


def _simulate(programs, n: int, backend: str, policy, device):
    if backend == "dense":
        return DenseBatch(len(programs), n, device=device).run(programs)
    return simulate_batch(programs, n, policy, device=device)


def _parity_value(counts: dict[str, int], support: list[int], shots: int) -> float:
    total = 0
    for bits, count in counts.items():
        parity = sum(int(bits[q]) for q in support) % 2
        total += count if parity == 0 else -count
    return total / shots


def grid_energies(ansatz, thetas, hamiltonian, backend: str = "mps",
                  policy: TruncationPolicy | None = None, shots: int | None = None,
                  seed: int | None = None, *, device=None) -> list[float]:
    """``energy(ansatz, t, ...)`` for every t in ``thetas``, batched on the GPU."""
    _check_backend(backend)
    programs = [_unitary_program(ansatz, float(t)) for t in thetas]
    return _program_energies(programs, hamiltonian, backend, policy, shots, seed, device)


def parameter_energies(ansatz, parameter_vectors, hamiltonian, backend: str = "mps",
                       policy: TruncationPolicy | None = None, shots: int | None = None,
                       seed: int | None = None, *, device=None) -> list[float]:
    """Multi-parameter sweep: <H> for the ansatz with ALL its formal parameters bound
    to each vector of ``parameter_vectors`` (e.g. config 2's 80-angle vectors).

    The reference driver is single-parameter (``vqe.py:30-35``); this extends it
    with the same per-vector semantics -- ``bind_parameters`` positionally,
    ``flatten``, MEASUREs dropped, E = sum_k c_k <P_k> left to right (``vqe.py:87-89``)
    or the sampled estimate (``vqe.py:90-97``) -- with every vector one state of a
    shared batch. ``IrError`` if a vector's length differs from the formal count."""
    _check_backend(backend)
    programs = [_bound_program(ansatz, vec) for vec in parameter_vectors]
    return _program_energies(programs, hamiltonian, backend, policy, shots, seed, device)


def _program_energies(programs, hamiltonian, backend, policy, shots, seed, device) -> list[float]:
    n = hamiltonian.n
    terms = [(float(c), str(p)) for c, p in hamiltonian.terms]
    for prog in programs:
        if num_qubits(prog) > n:
            raise ValueError(f"ansatz touches qubit {num_qubits(prog) - 1}, "
                             f"Hamiltonian has {n} qubit(s)")
    if shots is None:
        out: list[float] = []
        paulis = [p for _, p in terms]
        coeffs = [c for c, _ in terms]
        for a in range(0, len(programs), _MAX_STATES_PER_BATCH):
            batch = _simulate(programs[a:a + _MAX_STATES_PER_BATCH], n, backend, policy, device)
            out.extend(float(e) for e in batch_energies(batch, paulis, coeffs))
        return out
    # sampled: one state per (grid point, non-identity term)
    jobs = [(v, k) for v in range(len(programs)) for k, (_, p) in enumerate(terms)
            if set(p) != {"I"}]
    parity = {}
    for a in range(0, len(jobs), _MAX_STATES_PER_BATCH):
        chunk = jobs[a:a + _MAX_STATES_PER_BATCH]
        progs = [programs[v] + _basis_rotations(terms[k][1]) for v, k in chunk]
        batch = _simulate(progs, n, backend, policy, device)
        for s, (v, k) in enumerate(chunk):
            rng = np.random.default_rng([0 if seed is None else seed, k])
            counts = batch.sample(s, shots, rng)
            support = [q for q, label in enumerate(terms[k][1]) if label != "I"]
            parity[v, k] = _parity_value(counts, support, shots)
    out = []
    for v in range(len(programs)):
        value = 0.0
        for k, (c, p) in enumerate(terms):
            value += c if set(p) == {"I"} else c * parity[v, k]
        out.append(value)
    return out


def energy(ansatz, theta: float, hamiltonian, backend: str = "mps",
           policy: TruncationPolicy | None = None, shots: int | None = None,
           seed: int | None = None, *, device=None) -> float:
    """<psi(theta)|H|psi(theta)> for the bound ansatz (``vqe.py:70-97``)."""
    return grid_energies(ansatz, [theta], hamiltonian, backend, policy, shots, seed,
                         device=device)[0]


def sweep(ansatz, hamiltonian, start: float = -pi, stop: float = pi, count: int = 100,
          backend: str = "mps", policy: TruncationPolicy | None = None,
          shots: int | None = None, seed: int | None = None, *, device=None) -> SweepResult:
    """Uniform inclusive grid scan, argmin ties toward smaller theta (``vqe.py:100-125``)."""
    if count < 2:
        raise ValueError("grid needs at least 2 points")
    thetas = np.linspace(start, stop, count)
    energies_ = grid_energies(ansatz, [float(t) for t in thetas], hamiltonian, backend,
                              policy, shots, seed, device=device)
    best = int(np.argmin(energies_))
    return SweepResult(thetas=tuple(float(t) for t in thetas), energies=tuple(energies_),
                       argmin_theta=float(thetas[best]), min_energy=float(energies_[best]))


def binomial_sigma(expectation: float, shots: int) -> float:
    """Standard error of a parity estimate at ``shots`` samples (``vqe.py:128-131``)."""
    return sqrt(max(0.0, 1.0 - expectation ** 2) / shots)
