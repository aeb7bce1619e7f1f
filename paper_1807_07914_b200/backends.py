"""Execution contract for the MPS backend (``R:src/mpsqvm/backends.py:47-79``).

``mps_run`` / ``run_program`` keep the reference signatures and semantics
(MEASURE skipped, register-size check, backend string). Programs run through
the layered GPU executor instead of a per-gate Python loop.
``simulate_batch`` is the batched entry point: many independent programs on
one device in shared launches (circuits / parameter vectors are
the natural shard).
"""

from __future__ import annotations

from .engine import MpsBatch, compile_batch
from .ir import num_qubits
from .mps import MpsState
from .policy import TruncationPolicy

BACKENDS = ("mps",)


def mps_run(program, n: int, policy: TruncationPolicy | None = None, *, device=None) -> MpsState:
    """Apply every unitary gate in order on a fresh MPS; MEASUREs are skipped."""
    state = MpsState(n, policy, device=device)
    state._batch.execute(compile_batch([program], n))
    return state


def run_program(program, n: int | None = None, backend: str = "mps",
                policy: TruncationPolicy | None = None, *, device=None) -> MpsState:
    if n is None:
        n = num_qubits(program)
    elif n < num_qubits(program):
        raise ValueError(f"program touches qubit {num_qubits(program) - 1}, register has {n}")
    if backend == "mps":
        return mps_run(program, n, policy, device=device)
    raise ValueError(f"unknown backend {backend!r}; expected one of {BACKENDS} "
                     "(the dense oracle is out of scope for this framework)")


def simulate_batch(programs, n: int, policy: TruncationPolicy | None = None, *, device=None,
                   mode: int = 0) -> MpsBatch:
    """Run ``programs[i]`` on state i of a fresh ``MpsBatch`` (one device)."""
    batch = MpsBatch(len(programs), n, policy, device=device)
    batch.execute(compile_batch(programs, n), mode=mode)
    return batch
