"""Execution contract for the MPS backend (``R:src/mpsqvm/backends.py:47-79``).

``mps_run`` / ``run_program`` keep the reference signatures and semantics
(MEASURE skipped, register-size check, backend string; ``backend="dense"`` is
the GPU statevector of ``dense.py``). Programs run through the layered GPU
executor instead of a per-gate Python loop.
``simulate_batch`` is the batched entry point: many independent programs on
one device in shared launches (circuits / parameter vectors are
the natural shard).
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from .dense import DenseState, dense_run
from .engine import MpsBatch, compile_batch
from .ir import num_qubits
from .mps import MpsState
from .policy import TruncationPolicy

BACKENDS = ("mps", "dense")


def mps_run(program, n: int, policy: TruncationPolicy | None = None, *, device=None) -> MpsState:
    """Apply every unitary gate in order on a fresh MPS; MEASUREs are skipped."""
    state = MpsState(n, policy, device=device)
    state._batch.execute(compile_batch([program], n))
    return state


def run_program(program, n: int | None = None, backend: str = "mps",
                policy: TruncationPolicy | None = None, *, device=None) -> MpsState | DenseState:
    if n is None:
        n = num_qubits(program)
    elif n < num_qubits(program):
        raise ValueError(f"program touches qubit {num_qubits(program) - 1}, register has {n}")
    if backend == "mps":
        return mps_run(program, n, policy, device=device)
    if backend == "dense":
        return dense_run(program, n, device=device)
    raise ValueError(f"unknown backend {backend!r}; expected one of {BACKENDS}")


def simulate_batch(programs, n: int, policy: TruncationPolicy | None = None, *, device=None,
                   mode: int = 0, chunk: int | None = None, keep_records: bool = False) -> MpsBatch:
    """Run ``programs[i]`` on state i of a fresh ``MpsBatch`` (one device).

    Batches of 256 or more circuits are planned and launched in ``chunk``-circuit
    slices (default: a quarter of the batch, at least 128): launches are asynchronous,
    so the host plans slice k+1 -- the one per-op host cost -- while the GPU runs
    slice k. Each state's program lies in one slice, so results are those of one plan
    (bit-identical). cfg4 (measured, B200): 256 circuits 262 -> 303 circuits/s,
    1024 circuits 280 -> 334 circuits/s (``tools/cfg4_chunks.py``).
    """
    S = len(programs)
    batch = MpsBatch(S, n, policy, device=device, keep_records=keep_records)
    if chunk is None:
        chunk = S if S < 256 else max(128, -(-S // 4))
    for c0 in range(0, S, max(1, chunk)):
        c1 = min(S, c0 + chunk)
        batch.execute(compile_batch(programs[c0:c1], n, states=range(c0, c1)), mode=mode)
    return batch


@dataclass
class RunRecord:
    """Results of one program execution (``backends.py:25-44``)."""

    counts: dict[str, int] = field(default_factory=dict)
    max_bond_seen: int | None = None
    memory_estimate_bytes: int = 0
    trunc_error_sq: float = 0.0
    wall_time: float = 0.0

    def to_json_dict(self, include_wall_time: bool = True) -> dict:
        out = {"counts": self.counts, "max_bond_seen": self.max_bond_seen,
               "memory_estimate_bytes": self.memory_estimate_bytes,
               "trunc_error_sq": self.trunc_error_sq}
        if include_wall_time:
            out["wall_time"] = self.wall_time
        return out


def measured_qubits(program) -> list[int]:
    """Qubits of the MEASURE instructions, in program order (``backends.py:82-84``)."""
    return [i.qubits[0] for i in program
            if getattr(i, "kind", None) is not None and i.kind.value == "MEASURE"]


def execute(program, n: int | None = None, backend: str = "mps",
            policy: TruncationPolicy | None = None, shots: int = 1024,
            seed: int | None = None, *, device=None) -> RunRecord:
    """Run, sample the measured qubits on the GPU, collect stats (``backends.py:87-113``)."""
    start = time.perf_counter()
    state = run_program(program, n, backend, policy, device=device)
    if isinstance(state, MpsState):
        record = RunRecord(max_bond_seen=state.max_bond_seen,
                           memory_estimate_bytes=state.memory_estimate_bytes(),
                           trunc_error_sq=state.trunc_error_sq)
    else:
        record = RunRecord(memory_estimate_bytes=16 * 2 ** state.n)
    targets = measured_qubits(program)
    if targets and shots > 0:
        full = state.sample(shots, np.random.default_rng(seed))
        for bits, count in sorted(full.items()):
            key = "".join(bits[q] for q in targets)
            record.counts[key] = record.counts.get(key, 0) + count
    record.wall_time = time.perf_counter() - start
    return record
