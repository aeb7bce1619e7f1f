"""Drop-in ``MpsState`` surface beyond the config paths: conditional_prob_zero
(R:src/mpsqvm/mps.py:206-214), the per-gate call path the reference's own
callers use (R:src/mpsqvm/bench.py:99-108, tests/test_acceptance.py:61-73),
capacity sized from the true bond dimensions, and device placement."""

import numpy as np
import pytest
import torch

from conftest import assert_scaled_close

pytestmark = pytest.mark.gpu

from oracle.mps_oracle import oracle_run
from paper_1807_07914_b200 import (GateKind, Instruction, MpsBatch, MpsState, TruncationPolicy, gate_matrix,
                                   mps_run)
from paper_1807_07914_b200.workloads import brick_circuit, random_program


def test_conditional_prob_zero_chain_matches_oracle():
    """Walk a prefix down the chain like MpsState.sample does (mps.py:216-237), each
    side with its own successor vectors: the conditional probabilities and the
    successor norms are gauge-invariant and must agree (the vectors themselves carry
    the Vidal gauge of each implementation's singular vectors, like Gamma)."""
    rng = np.random.default_rng(5)
    n = 10
    prog = brick_circuit(n, 6, rng)
    st = mps_run(prog, n, TruncationPolicy(1e-10, 16))
    o = oracle_run(prog, n, 1e-10, 16)
    vec = np.ones(1, dtype=complex)
    ref = np.ones(1, dtype=complex)
    for k in range(n):
        p0, w0, w1 = st.conditional_prob_zero(vec, k)
        t = o.site_matrix(k)
        r0, r1 = ref @ t[:, 0, :], ref @ t[:, 1, :]
        a, b = float(np.vdot(r0, r0).real), float(np.vdot(r1, r1).real)
        rp = a / (a + b) if a + b > 0 else 0.5
        assert abs(p0 - rp) <= 1e-12, (k, p0, rp)
        assert abs(np.linalg.norm(w0) - np.linalg.norm(r0)) <= 1e-12 * max(1.0, np.linalg.norm(r0))
        assert abs(np.linalg.norm(w1) - np.linalg.norm(r1)) <= 1e-12 * max(1.0, np.linalg.norm(r1))
        if rng.random() < p0:
            vec, ref = w0, r0
        else:
            vec, ref = w1, r1
    with pytest.raises(ValueError):
        st.conditional_prob_zero(np.ones(3), 0)


def test_conditional_prob_zero_vanishing_branch_is_half():
    st = MpsState(2)                       # |00>: w1 = 0 at site 0, p0 = 1
    p0, w0, w1 = st.conditional_prob_zero(np.zeros(1, complex), 0)
    assert p0 == 0.5 and not w0.any() and not w1.any()


def test_per_gate_calls_equal_layered_run_bit_for_bit():
    """MpsState.apply_* one gate at a time (no planner, pinned staging ring) and the
    layered executor perform the same per-op arithmetic: identical bits."""
    rng = np.random.default_rng(21)
    n = 9
    prog = random_program(n, 160, rng)
    a = MpsState(n, TruncationPolicy(1e-8, 12))
    for op in prog:
        g = gate_matrix(op)
        if len(op.qubits) == 1:
            a.apply_one_qubit(g, op.qubits[0])
        elif abs(op.qubits[0] - op.qubits[1]) == 1 and op.qubits[0] < op.qubits[1]:
            a.apply_two_qubit_adjacent(g, op.qubits[0])
        else:
            a.apply_two_qubit_routed(g, op.qubits[0], op.qubits[1])
    b = mps_run(prog, n, TruncationPolicy(1e-8, 12))
    a.synchronize()
    np.testing.assert_array_equal(a._batch.host_dims(), b._batch.host_dims())
    np.testing.assert_array_equal(a._batch.lam.cpu().numpy(), b._batch.lam.cpu().numpy())
    np.testing.assert_array_equal(a._batch.gamma.cpu().numpy(), b._batch.gamma.cpu().numpy())
    assert a.trunc_error_sq == b.trunc_error_sq
    assert a.peak_entries == b.peak_entries and a.max_bond_seen == b.max_bond_seen
    # the per-gate path retains only the latest update record (bounded memory)
    assert len(a._batch._logs) <= 1


def test_per_gate_errors_keep_reference_messages():
    st = MpsState(4)
    with pytest.raises(ValueError, match="out of range"):
        st.apply_one_qubit(np.eye(2), 4)
    with pytest.raises(ValueError, match="no right neighbour"):
        st.apply_two_qubit_adjacent(np.eye(4), 3)
    with pytest.raises(ValueError, match="distinct"):
        st.apply_two_qubit_routed(np.eye(4), 1, 1)
    with pytest.raises(ValueError, match="not unitary"):
        st.apply_one_qubit(np.ones((2, 2)), 0)


def test_capacity_follows_true_bond_dimensions():
    """with the default policy (cutoff 1e-4, no max_bond) a deep CNOT-only
    circuit on |0...0> keeps every bond at 1; the host's doubling bound would pass
    1024 after 11 layers. Capacity must follow the real bonds, not the bound."""
    n = 26
    prog = []
    for d in range(30):
        prog += [Instruction(GateKind.CNOT, (a, a + 1)) for a in range(d % 2, n - 1, 2)]
    st = mps_run(prog, n)
    assert st.max_bond() == 1 and st.max_bond_seen == 1
    assert st._batch.cap <= 2
    assert st.amplitude("0" * n) == 1.0


def test_keep_records_retains_every_plan():
    rng = np.random.default_rng(2)
    b = MpsBatch(1, 8, TruncationPolicy(1e-10, 8), keep_records=True)
    for _ in range(3):
        b.run([brick_circuit(8, 2, rng)])
    rec = b.update_records(0)
    assert len(rec) == 3 * 7 and len(b._logs) == 3
    assert np.all(rec["margin"] > 0) and np.all(rec["gap"] >= 0)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs")
def test_state_on_second_device():
    prog = brick_circuit(10, 6, np.random.default_rng(3))
    a = mps_run(prog, 10, TruncationPolicy(1e-10, 16), device="cuda:1")
    b = mps_run(prog, 10, TruncationPolicy(1e-10, 16), device="cuda:0")
    assert a._batch.gamma.device.index == 1
    np.testing.assert_array_equal(a._batch.lam.cpu().numpy(), b._batch.lam.cpu().numpy())
