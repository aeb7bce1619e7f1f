"""GPU dense statevector backend: drop-in for ``R:src/mpsqvm/dense.py``.

The reference's dense simulator is the SVD-free oracle the MPS backend is
checked against (and ``backend="dense"`` of ``run_program`` / ``execute`` /
``vqe.sweep``). Here the 2^n complex128 amplitudes live in HBM and every
operation is a ``libbmps.so`` kernel (``csrc/bmps_dense.cuh``): per-gate
coalesced streaming passes, a shared-memory-resident whole-program kernel for
n <= 12, a fused Pauli-string expectation pass, and a marginal-probability heap
for the sequential conditional sampler (same uniform stream as the reference,
so seeded counts agree). There is no CPU fallback.

Public surface as in the reference (``dense.py:16-131``): ``DenseState`` with
``amps`` (host copy on read, uploaded on assignment), ``apply_one_qubit``,
``apply_two_qubit``, ``amplitude``, ``norm_sq``, ``expectation_pauli``,
``distribution``, ``conditional_prob_zero``, ``sample``; ``dense_run``,
``dense_expectation``, ``dense_distribution``, ``oracle_qubit_cap`` (same
``MPSQVM_ORACLE_QUBIT_CAP`` variable and default 24, so the reference's cap
semantics and error messages carry over; raise it up to 33 on a B200).
"""

from __future__ import annotations

import os

import numpy as np
import torch

from . import _native
from .engine import _stream, require_cuda
from .gates import check_unitary, gate_matrix

DEFAULT_QUBIT_CAP = 24
MAX_QUBITS = 33        # kDenseMaxQubits: 128 GB of amplitudes
SMEM_QUBITS = 12       # kDenseSmemQubits: whole-program kernel threshold


def oracle_qubit_cap() -> int:
    return int(os.environ.get("MPSQVM_ORACLE_QUBIT_CAP", DEFAULT_QUBIT_CAP))


def _pauli_masks(pauli: str, n: int) -> tuple[int, int, int]:
    """(x mask, sign mask, #Y) with qubit q at bit n-1-q (dense.py:23)."""
    xm = zm = ny = 0
    for q, ch in enumerate(pauli):
        b = 1 << (n - 1 - q)
        if ch == "X":
            xm |= b
        elif ch == "Y":
            xm |= b
            zm |= b
            ny += 1
        elif ch == "Z":
            zm |= b
        elif ch != "I":
            raise ValueError(f"bad Pauli label {ch!r} in {pauli!r}")
    return xm, zm, ny


class DenseState:
    """Full 2^n amplitude vector in HBM; flat index has qubit 0 as the high bit."""

    def __init__(self, n: int, *, device=None):
        cap = oracle_qubit_cap()
        if not 1 <= n <= cap:
            raise ValueError(f"dense oracle supports 1..{cap} qubits, got {n}")
        if n > MAX_QUBITS:
            raise ValueError(f"dense backend supports at most {MAX_QUBITS} qubits on one device, got {n}")
        self.n = n
        self.device = require_cuda(device)
        self.lib = _native.load()
        with torch.cuda.device(self.device):
            self._amps = torch.empty(2 ** n, dtype=torch.complex128, device=self.device)
            _native.check(self.lib.bmps_dense_init(self._amps.data_ptr(), 1, n, _stream()),
                          "bmps_dense_init")
        self._tree = None      # marginal-probability heap, built lazily per state version
        self._tree_valid = False

    # -- amplitudes ------------------------------------------------------------
    @property
    def amps(self) -> np.ndarray:
        return self._amps.cpu().numpy()

    @amps.setter
    def amps(self, value) -> None:
        v = np.ascontiguousarray(value, dtype=np.complex128).reshape(-1)
        if v.size != 2 ** self.n:
            raise ValueError(f"need {2 ** self.n} amplitudes, got {v.size}")
        self._amps.copy_(torch.from_numpy(v))
        self._tree_valid = False

    @property
    def amps_device(self) -> torch.Tensor:
        """The device buffer itself (complex128 [2^n], no copy)."""
        return self._amps

    # -- gates -------------------------------------------------------------------
    def _check_qubits(self, qubits) -> None:
        for q in qubits:
            if not 0 <= q < self.n:
                raise ValueError(f"qubit {q} out of range for {self.n} qubits")

    def apply_one_qubit(self, gate: np.ndarray, q: int) -> None:
        self._check_qubits((q,))
        check_unitary(gate)
        g = np.ascontiguousarray(gate, dtype=np.complex128)
        with torch.cuda.device(self.device):
            rc = self.lib.bmps_dense_apply_1q(self._amps.data_ptr(), self.n, q, g.ctypes.data, _stream())
        _native.check(rc, "bmps_dense_apply_1q")
        self._tree_valid = False

    def apply_two_qubit(self, gate: np.ndarray, q1: int, q2: int) -> None:
        self._check_qubits((q1, q2))
        if q1 == q2:
            raise ValueError("two-qubit gate needs two distinct qubits")
        check_unitary(gate)
        g = np.ascontiguousarray(gate, dtype=np.complex128)
        with torch.cuda.device(self.device):
            rc = self.lib.bmps_dense_apply_2q(self._amps.data_ptr(), self.n, q1, q2, g.ctypes.data,
                                              _stream())
        _native.check(rc, "bmps_dense_apply_2q")
        self._tree_valid = False

    def run(self, program) -> "DenseState":
        """Apply a whole program (MEASURE skipped): one shared-memory kernel for
        n <= 12, per-gate streaming passes above."""
        ops, mats = _lower(program, self.n)
        if not ops:
            return self
        if self.n <= SMEM_QUBITS:
            _run_smem(self.lib, self._amps, 1, self.n, [ops], [mats], self.device)
        else:
            for (ar, q1, q2), m in zip(ops, mats):
                if ar == 1:
                    self.apply_one_qubit(m, q1)
                else:
                    self.apply_two_qubit(m, q1, q2)
        self._tree_valid = False
        return self

    # -- queries -----------------------------------------------------------------
    def amplitude(self, bits: str) -> complex:
        if len(bits) != self.n or any(b not in "01" for b in bits):
            raise ValueError(f"need a bitstring of length {self.n}, got {bits!r}")
        return complex(self._amps[int(bits, 2)].item())

    def norm_sq(self) -> float:
        return float(self._expect_raw(["I" * self.n])[0].real)

    def expectation_pauli(self, pauli: str) -> float:
        if len(pauli) != self.n:
            raise ValueError(f"Pauli string length {len(pauli)} != qubit count {self.n}")
        value = complex(self._expect_raw([pauli])[0])
        if abs(value.imag) > 1e-10:
            raise RuntimeError(f"expectation has imaginary residue {value.imag:.3e}")
        return value.real

    def expectations_pauli(self, paulis) -> np.ndarray:
        """Batched ``expectation_pauli`` (one fused pass per string, one launch)."""
        for p in paulis:
            if len(p) != self.n:
                raise ValueError(f"Pauli string length {len(p)} != qubit count {self.n}")
        vals = self._expect_raw(list(paulis))
        bad = np.abs(vals.imag) > 1e-10
        if bad.any():
            raise RuntimeError(f"expectation has imaginary residue {vals.imag[bad][0]:.3e}")
        return vals.real.copy()

    def _expect_raw(self, paulis: list[str]) -> np.ndarray:
        return _expect(self.lib, self._amps, 1, self.n, np.zeros(len(paulis), np.int32), paulis,
                       self.device)

    def distribution(self) -> dict[str, float]:
        """Exact |amplitude|^2 per basis bitstring."""
        probs = (self._amps.abs() ** 2).cpu().numpy()
        return {format(i, f"0{self.n}b"): float(p) for i, p in enumerate(probs)}

    def _prob_tree(self) -> torch.Tensor:
        if self._tree is None:
            self._tree = torch.empty(2 ** (self.n + 1), dtype=torch.float64, device=self.device)
        if not self._tree_valid:
            with torch.cuda.device(self.device):
                rc = self.lib.bmps_dense_prob_tree(self._amps.data_ptr(), self.n, self._tree.data_ptr(),
                                                   _stream())
            _native.check(rc, "bmps_dense_prob_tree")
            self._tree_valid = True
        return self._tree

    def conditional_prob_zero(self, prefix_bits: str, k: int) -> float:
        """P(qubit k = 0 | qubits 0..k-1 fixed to prefix_bits) (dense.py:88-96)."""
        if len(prefix_bits) != k or not 0 <= k < self.n:
            raise ValueError(f"need a prefix of length k for 0 <= k < {self.n}")
        node = (1 << k) + (int(prefix_bits, 2) if k else 0)
        pair = self._prob_tree()[2 * node:2 * node + 2].cpu().numpy()
        total = pair[0] + pair[1]
        return float(pair[0] / total) if total > 0 else 0.5

    def sample(self, shots: int, rng: np.random.Generator) -> dict[str, int]:
        """Sequential conditional sampling, RNG-compatible with the MPS path (dense.py:98-110)."""
        if shots < 1:
            raise ValueError("shots must be >= 1")
        tree = self._prob_tree()
        u = torch.from_numpy(rng.random((shots, self.n))).to(self.device)
        out = torch.empty(shots, dtype=torch.int64, device=self.device)
        with torch.cuda.device(self.device):
            rc = self.lib.bmps_dense_sample(tree.data_ptr(), self.n, u.data_ptr(), shots, out.data_ptr(),
                                            _stream())
        _native.check(rc, "bmps_dense_sample")
        idx, cnt = np.unique(out.cpu().numpy(), return_counts=True)
        return {format(int(i), f"0{self.n}b"): int(c) for i, c in zip(idx, cnt)}


def _lower(program, n: int):
    ops, mats = [], []
    for instr in program:
        kind = getattr(instr, "kind", None)
        if kind is not None and kind.value == "MEASURE":
            continue
        for q in instr.qubits:
            if not 0 <= q < n:
                raise ValueError(f"qubit {q} out of range for {n} qubits")
        m = np.asarray(gate_matrix(instr), dtype=np.complex128)
        if len(instr.qubits) == 1:
            ops.append((1, instr.qubits[0], 0))
        else:
            if instr.qubits[0] == instr.qubits[1]:
                raise ValueError("two-qubit gate needs two distinct qubits")
            ops.append((2, instr.qubits[0], instr.qubits[1]))
        mats.append(m)
    return ops, mats


def _run_smem(lib, amps: torch.Tensor, S: int, n: int, ops_list, mats_list, device) -> None:
    """All S states (amps [S, 2^n]) through their own equal-length gate lists."""
    nops = len(ops_list[0])
    ops = np.zeros((S, nops, 3), np.int32)
    mats = np.zeros((S, nops, 16), np.complex128)
    for s in range(S):
        if len(ops_list[s]) != nops:
            raise ValueError("batched dense programs must have equal gate counts")
        ops[s] = np.asarray(ops_list[s], np.int32).reshape(nops, 3)
        for k, m in enumerate(mats_list[s]):
            mats[s, k, :m.size] = m.reshape(-1)
    d_ops = torch.from_numpy(ops).to(device)
    d_mats = torch.from_numpy(mats).to(device)
    with torch.cuda.device(device):
        rc = lib.bmps_dense_run_smem(amps.data_ptr(), S, n, d_ops.data_ptr(), d_mats.data_ptr(), nops,
                                     _stream())
    _native.check(rc, "bmps_dense_run_smem")


def _expect(lib, amps: torch.Tensor, S: int, n: int, state_idx: np.ndarray, paulis, device) -> np.ndarray:
    K = len(paulis)
    if K == 0:
        return np.zeros(0, np.complex128)
    masks = np.zeros((K, 2), np.uint64)
    ny = np.zeros(K, np.int32)
    for k, p in enumerate(paulis):
        xm, zm, y = _pauli_masks(p, n)
        masks[k] = (xm, zm)
        ny[k] = y
    d_idx = torch.from_numpy(np.ascontiguousarray(state_idx, np.int32)).to(device)
    d_masks = torch.from_numpy(masks.view(np.int64)).to(device)
    d_ny = torch.from_numpy(ny).to(device)
    wsb = lib.bmps_dense_expect_workspace_bytes(K)
    ws = torch.empty(max(wsb // 8, 1), dtype=torch.float64, device=device)
    out = torch.empty(K, dtype=torch.complex128, device=device)
    with torch.cuda.device(device):
        rc = lib.bmps_dense_expect(amps.data_ptr(), S, n, d_idx.data_ptr(), d_masks.data_ptr(),
                                   d_ny.data_ptr(), K, ws.data_ptr(), wsb, out.data_ptr(), _stream())
    _native.check(rc, "bmps_dense_expect")
    return out.cpu().numpy()


class DenseBatch:
    """S independent dense states of n qubits in one buffer (the ``backend="dense"``
    VQE-sweep path: every grid point is one state, all evolved in one launch)."""

    def __init__(self, S: int, n: int, *, device=None):
        cap = oracle_qubit_cap()
        if not 1 <= n <= cap:
            raise ValueError(f"dense oracle supports 1..{cap} qubits, got {n}")
        self.S, self.n = S, n
        self.device = require_cuda(device)
        self.lib = _native.load()
        with torch.cuda.device(self.device):
            self.amps = torch.empty((S, 2 ** n), dtype=torch.complex128, device=self.device)
            _native.check(self.lib.bmps_dense_init(self.amps.data_ptr(), S, n, _stream()), "bmps_dense_init")

    def run(self, programs) -> "DenseBatch":
        lowered = [_lower(p, self.n) for p in programs]
        if len(lowered) != self.S:
            raise ValueError(f"need {self.S} programs, got {len(lowered)}")
        counts = {len(o) for o, _ in lowered}
        if self.n <= SMEM_QUBITS and len(counts) == 1:
            if counts.pop():
                _run_smem(self.lib, self.amps, self.S, self.n, [o for o, _ in lowered],
                          [m for _, m in lowered], self.device)
            return self
        for s, (ops, mats) in enumerate(lowered):
            ptr = self.amps[s].data_ptr()
            with torch.cuda.device(self.device):
                for (ar, q1, q2), m in zip(ops, mats):
                    m = np.ascontiguousarray(m)
                    if ar == 1:
                        rc = self.lib.bmps_dense_apply_1q(ptr, self.n, q1, m.ctypes.data, _stream())
                    else:
                        rc = self.lib.bmps_dense_apply_2q(ptr, self.n, q1, q2, m.ctypes.data, _stream())
                    _native.check(rc, "bmps_dense_apply")
        return self

    def expectations(self, state_idx, paulis) -> np.ndarray:
        """<P_k> of state state_idx[k] (real parts; imaginary residue checked)."""
        vals = _expect(self.lib, self.amps, self.S, self.n, np.asarray(state_idx, np.int32), list(paulis),
                       self.device)
        bad = np.abs(vals.imag) > 1e-10
        if bad.any():
            raise RuntimeError(f"expectation has imaginary residue {vals.imag[bad][0]:.3e}")
        return vals.real.copy()

    def sample(self, s: int, shots: int, rng: np.random.Generator) -> dict[str, int]:
        return self.state(s).sample(shots, rng)

    def state(self, s: int) -> DenseState:
        """A ``DenseState`` view sharing state ``s``'s amplitudes."""
        st = DenseState.__new__(DenseState)
        st.n, st.device, st.lib = self.n, self.device, self.lib
        st._amps = self.amps[s]
        st._tree, st._tree_valid = None, False
        return st


def dense_run(program, n: int, *, device=None) -> DenseState:
    """Apply every unitary gate of the program in order; MEASUREs are skipped (dense.py:112-123)."""
    return DenseState(n, device=device).run(program)


def dense_expectation(state: DenseState, pauli: str) -> float:
    return state.expectation_pauli(pauli)


def dense_distribution(state: DenseState) -> dict[str, float]:
    return state.distribution()
