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

    Batches of 256 or more circuits are planned and launched in slices: launches are
    asynchronous, so the host plans slice k+1 -- the one per-op host cost -- while the
    GPU runs slice k. Only the first slice's planning is exposed, so the default
    schedule starts small and doubles (S/16, S/8, then quarters of the batch; at least
    64 circuits); ``chunk`` forces equal slices. Each state's program lies in one
    slice, so results are those of one plan (bit-identical). cfg4 (measured, B200):
    1024 circuits 280 (one plan) -> 334 (quarters) circuits/s (``tools/cfg4_chunks.py``).
    """
    S = len(programs)
    batch = MpsBatch(S, n, policy, device=device, keep_records=keep_records)
    for c0, c1 in slice_schedule(S, chunk):
        batch.execute(compile_batch(programs[c0:c1], n, states=range(c0, c1)), mode=mode)
    return batch


def slice_schedule(S: int, chunk: int | None = None) -> list[tuple[int, int]]:
    """[c0, c1) circuit slices of ``simulate_batch``: equal ``chunk``-sized ones, or by
    default one slice below 256 circuits, else S/16, S/8, then quarters (>= 64 each; a
    remainder under half a slice joins the last one)."""
    if chunk is not None:
        chunk = max(1, chunk)
        return [(c0, min(S, c0 + chunk)) for c0 in range(0, S, chunk)]
    if S < 256:
        return [(0, S)] if S else []
    sizes, left, step = [], S, max(64, S // 16)
    cap = max(64, -(-S // 4))
    while left > 0:
        take = min(step, left)
        sizes.append(take)
        left -= take
        step = min(cap, step * 2)
    if len(sizes) > 1 and sizes[-1] < cap // 2:
        last = sizes.pop()
        sizes[-1] += last
    out, c0 = [], 0
    for z in sizes:
        out.append((c0, c0 + z))
        c0 += z
    return out


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
