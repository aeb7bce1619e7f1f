"""B200-native matrix-product-state simulator (drop-in for the mpsqvm MPS backend).

Public names mirror the reference package's MPS hot path
(``R:src/mpsqvm/__init__.py``): ``MpsState``, ``TruncationPolicy``, ``mps_run``,
``run_program``, ``GateKind``, ``Instruction``, ``PauliHamiltonian``, and the
dense statevector backend (``DenseState``, ``dense_run``, ...). Compute
runs in ``libbmps.so`` (hand-written sm_100a CUDA behind the C ABI in
``include/bmps.h``); there is no CPU fallback.
"""

from .backends import BACKENDS, RunRecord, execute, measured_qubits, mps_run, run_program, simulate_batch
from .dense import DenseBatch, DenseState, dense_distribution, dense_expectation, dense_run
from .engine import MpsBatch, compile_batch
from .gates import SWAP_MATRIX, check_unitary, gate_matrix
from .hamiltonian import PauliHamiltonian, pauli_matrix
from .ir import (CompositeInstruction, GateKind, Instruction, IrError, MatrixGate, bind_parameters,
                 flatten, num_qubits)
from .mps import MpsState
from .policy import TruncationPolicy

__all__ = [
    "BACKENDS", "DenseBatch", "DenseState", "dense_distribution", "dense_expectation", "dense_run", "CompositeInstruction", "bind_parameters", "flatten", "RunRecord", "execute", "measured_qubits", "GateKind", "Instruction", "IrError", "MatrixGate", "MpsBatch", "MpsState",
    "PauliHamiltonian", "SWAP_MATRIX", "TruncationPolicy", "check_unitary", "compile_batch",
    "gate_matrix", "mps_run", "num_qubits", "pauli_matrix", "run_program", "simulate_batch",
]
