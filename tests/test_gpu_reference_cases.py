"""Known-answer cases of the reference suite (R:tests/test_mps.py), on the GPU path."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_1807_07914_b200 import GateKind, Instruction, MpsState, TruncationPolicy, gate_matrix, mps_run
from paper_1807_07914_b200.workloads import random_program

EXACT = TruncationPolicy(cutoff=0.0)
H = gate_matrix(Instruction(GateKind.H, (0,)))
X = gate_matrix(Instruction(GateKind.X, (0,)))
CNOT = gate_matrix(Instruction(GateKind.CNOT, (0, 1)))


def bell():
    return [Instruction(GateKind.H, (0,)), Instruction(GateKind.CNOT, (0, 1))]


def ghz3():
    return bell() + [Instruction(GateKind.CNOT, (1, 2))]


def test_product_state_amplitudes():  # test_mps.py:18-23
    st = MpsState(3)
    for bits in ["000", "001", "010", "100", "111"]:
        assert st.amplitude(bits) == pytest.approx(1.0 if bits == "000" else 0.0)


def test_single_site_and_memory():  # test_mps.py:25-31
    st = MpsState(1)
    assert st.site_tensors[0].shape == (1, 2, 1)
    np.testing.assert_allclose(st.site_tensors[0].reshape(2), [1, 0])
    assert MpsState(85).memory_estimate_bytes() == 2720
    with pytest.raises(ValueError):
        MpsState(0)


def test_one_qubit_gates():  # test_mps.py:38-67
    st = MpsState(1)
    st.apply_one_qubit(X, 0)
    assert st.amplitude("1") == pytest.approx(1.0)
    st = MpsState(1)
    st.apply_one_qubit(H, 0)
    assert st.amplitude("0") == pytest.approx(2 ** -0.5)
    assert st.amplitude("1") == pytest.approx(2 ** -0.5)
    with pytest.raises(ValueError, match="unitary"):
        MpsState(2).apply_one_qubit(np.array([[1.0, 0.0], [0.0, 2.0]]), 0)
    with pytest.raises(ValueError):
        MpsState(2).apply_one_qubit(X, 2)


def test_bonds_untouched_by_1q(rng):  # test_mps.py:56-60
    st = mps_run(random_program(5, 20, rng), 5, EXACT)
    before = [len(v) for v in st.bond_vectors]
    st.apply_one_qubit(H, 2)
    assert [len(v) for v in st.bond_vectors] == before


def test_bell_schmidt_vector():  # test_mps.py:71-77
    st = MpsState(2, EXACT)
    st.apply_one_qubit(H, 0)
    st.apply_two_qubit_adjacent(CNOT, 0)
    np.testing.assert_allclose(st.bond_vectors[0], [2 ** -0.5] * 2, rtol=1e-12)
    assert st.amplitude("00") == pytest.approx(2 ** -0.5)
    assert st.amplitude("11") == pytest.approx(2 ** -0.5)


def test_product_in_product_out():  # test_mps.py:79-94
    st = MpsState(2, TruncationPolicy(1e-4))
    st.apply_one_qubit(X, 0)
    st.apply_two_qubit_adjacent(CNOT, 0)
    assert st.amplitude("11") == pytest.approx(1.0)
    assert st.max_bond() == 1
    st = MpsState(2, TruncationPolicy(1e-4))
    st.apply_one_qubit(H, 0)
    st.apply_two_qubit_adjacent(CNOT, 0)
    st.apply_two_qubit_adjacent(CNOT, 0)
    assert st.amplitude("00") == pytest.approx(2 ** -0.5)
    assert st.amplitude("10") == pytest.approx(2 ** -0.5)
    assert st.max_bond() == 1
    with pytest.raises(ValueError):
        MpsState(2).apply_two_qubit_adjacent(CNOT, 1)


def test_routing():  # test_mps.py:104-128, 157-159
    st = mps_run([Instruction(GateKind.X, (0,)), Instruction(GateKind.CNOT, (0, 2))], 3, EXACT)
    assert st.amplitude("101") == pytest.approx(1.0)
    st = mps_run([Instruction(GateKind.H, (0,)), Instruction(GateKind.CNOT, (0, 2))], 3, EXACT)
    assert st.amplitude("000") == pytest.approx(2 ** -0.5)
    assert st.amplitude("101") == pytest.approx(2 ** -0.5)
    st = mps_run([Instruction(GateKind.X, (2,)), Instruction(GateKind.CNOT, (2, 0))], 3, EXACT)
    assert st.amplitude("101") == pytest.approx(1.0)
    with pytest.raises(ValueError):
        MpsState(3).apply_two_qubit_routed(CNOT, 1, 1)


def test_queries():  # test_mps.py:163-187
    st = mps_run(ghz3(), 3, EXACT)
    assert st.amplitude("000") == pytest.approx(2 ** -0.5)
    assert st.amplitude("010") == pytest.approx(0.0)
    with pytest.raises(ValueError):
        MpsState(3).amplitude("01")
    st = mps_run(bell(), 2, EXACT)
    assert st.expectation_pauli("ZZ") == pytest.approx(1.0)
    assert st.expectation_pauli("ZI") == pytest.approx(0.0, abs=1e-12)
    assert st.expectation_pauli("XX") == pytest.approx(1.0)
    with pytest.raises(ValueError):
        st.expectation_pauli("Z")
    before = [t.copy() for t in st.site_tensors]
    st.expectation_pauli("XY")
    for old, new in zip(before, st.site_tensors):
        np.testing.assert_array_equal(old, new)


def test_bond_stats(rng):  # test_mps.py:224-231
    st = MpsState(10)
    assert st.max_bond() == 1
    assert st.memory_estimate_bytes() == 320
    assert mps_run(bell(), 2, EXACT).max_bond() == 2
    st = mps_run(random_program(10, 400, rng), 10, EXACT)
    assert st.max_bond_seen == 32


def test_norm_preserved_per_gate(rng):  # test_mps.py:235-244
    program = random_program(6, 40, rng)
    st = MpsState(6, EXACT)
    for instr in program:
        m = gate_matrix(instr)
        if instr.kind.num_qubits == 1:
            st.apply_one_qubit(m, instr.qubits[0])
        else:
            st.apply_two_qubit_routed(m, *instr.qubits)
        assert abs(st.norm_sq() - 1) < 1e-10


def test_storage_law(rng):  # test_mps.py:263-268
    for n in (6, 10):
        st = mps_run(random_program(n, 60, rng), n, EXACT)
        chi = st.max_bond_seen
        assert st.total_entries() <= n * 2 * chi ** 2 + (n - 1) * chi


def test_policy_keeps_at_least_one():  # test_mps.py:270-276
    st = MpsState(2, TruncationPolicy(cutoff=0.5, max_bond=1))
    st.apply_one_qubit(H, 0)
    st.apply_two_qubit_adjacent(CNOT, 0)
    assert st.max_bond() == 1
    assert st.trunc_error_sq == pytest.approx(0.5)
