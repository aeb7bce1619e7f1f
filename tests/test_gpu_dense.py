"""GPU dense statevector backend vs the reference semantics (R:tests/test_dense.py)
and the numpy dense oracle (oracle/dense_oracle.py, a restatement of
R:src/mpsqvm/dense.py): amplitudes / expectations to 1e-12 absolute (unit-norm
states), seeded sample counts identical to the reference's sequential sampler,
and the dense <-> MPS cross-checks the reference runs (R:tests/test_mps.py:127-152,
R:tests/test_cli.py:34-49, R:tests/test_acceptance.py:162-179)."""

import itertools

import numpy as np
import pytest

from conftest import assert_scaled_close

pytestmark = pytest.mark.gpu

from oracle.dense_oracle import dense_expectation as np_expectation
from oracle.dense_oracle import dense_run as np_dense_run
from paper_1807_07914_b200 import (DenseBatch, DenseState, GateKind, Instruction, PauliHamiltonian,
                                   TruncationPolicy, dense_distribution, dense_expectation,
                                   dense_run, execute, gate_matrix, mps_run, run_program)
from paper_1807_07914_b200.gates import rz
from paper_1807_07914_b200.vqe import sweep
from paper_1807_07914_b200.workloads import random_program

I = Instruction
EXACT = TruncationPolicy(cutoff=0.0)


def bell():
    return [I(GateKind.H, (0,)), I(GateKind.CNOT, (0, 1))]


def ghz3():
    return [I(GateKind.H, (0,)), I(GateKind.CNOT, (0, 1)), I(GateKind.CNOT, (1, 2))]


def random_paulis(n, count, rng):
    return ["".join("IXYZ"[int(v)] for v in rng.integers(0, 4, n)) for _ in range(count)]


def np_sample(psi, n, shots, rng):
    """The reference's DenseState.sample loop (dense.py:88-110), restated on numpy."""
    t = psi.reshape((2,) * n)
    counts = {}
    for _ in range(shots):
        bits = ""
        for k in range(n):
            block = t[tuple(int(b) for b in bits)]
            p0 = float(np.sum(np.abs(block[0]) ** 2))
            p1 = float(np.sum(np.abs(block[1]) ** 2))
            tot = p0 + p1
            bits += "0" if rng.random() < (p0 / tot if tot > 0 else 0.5) else "1"
        counts[bits] = counts.get(bits, 0) + 1
    return counts


# ---- R:tests/test_dense.py known answers -------------------------------------

def test_bell_amplitudes():
    np.testing.assert_allclose(dense_run(bell(), 2).amps, [2 ** -0.5, 0, 0, 2 ** -0.5], atol=1e-12)


def test_empty_program():
    np.testing.assert_allclose(dense_run([], 1).amps, [1, 0])


def test_qubit_out_of_range():
    with pytest.raises(ValueError):
        dense_run([I(GateKind.X, (3,))], 2)


def test_qubit_cap(monkeypatch):
    monkeypatch.setenv("MPSQVM_ORACLE_QUBIT_CAP", "4")
    with pytest.raises(ValueError, match="1..4"):
        DenseState(5)
    DenseState(4)


def test_measure_is_skipped():
    st = dense_run(bell() + [I(GateKind.MEASURE, (0,), (), 0)], 2)
    assert st.norm_sq() == pytest.approx(1.0)


def test_bell_zz_and_zero_state_x():
    assert dense_expectation(dense_run(bell(), 2), "ZZ") == pytest.approx(1.0)
    assert dense_expectation(dense_run([], 2), "XI") == pytest.approx(0.0, abs=1e-12)


def test_ghz_distribution():
    dist = dense_distribution(dense_run(ghz3(), 3))
    assert dist["000"] == pytest.approx(0.5) and dist["111"] == pytest.approx(0.5)
    assert sum(dist.values()) == pytest.approx(1.0)


def test_length_mismatch():
    with pytest.raises(ValueError):
        dense_expectation(dense_run([], 2), "Z")


def test_gate_algebra(rng):
    st = dense_run(random_program(3, 15, rng), 3)
    before = st.amps.copy()
    h = gate_matrix(I(GateKind.H, (0,)))
    st.apply_one_qubit(h, 1)
    st.apply_one_qubit(h, 1)
    np.testing.assert_allclose(st.amps, before, atol=1e-12)
    cnot = gate_matrix(I(GateKind.CNOT, (0, 1)))
    st.apply_two_qubit(cnot, 0, 2)
    st.apply_two_qubit(cnot, 0, 2)
    np.testing.assert_allclose(st.amps, before, atol=1e-12)


def test_rz_composition_up_to_phase(rng):
    st = dense_run(random_program(2, 15, rng), 2)
    a = st.amps.copy()
    st.apply_one_qubit(rz(0.4), 0)
    st.apply_one_qubit(rz(0.9), 0)
    combined = np.tensordot(rz(1.3), a.reshape(2, 2), axes=([1], [0]))
    assert abs(np.vdot(combined.reshape(-1), st.amps)) == pytest.approx(1.0)


def test_norm_preserved_per_gate(rng):
    st = DenseState(5)
    for instr in random_program(5, 30, rng):
        m = gate_matrix(instr)
        if len(instr.qubits) == 1:
            st.apply_one_qubit(m, instr.qubits[0])
        else:
            st.apply_two_qubit(m, *instr.qubits)
        assert abs(st.norm_sq() - 1) < 1e-10


# ---- parity with the numpy dense oracle ------------------------------------------

@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 12, 13, 16])
def test_amplitudes_and_paulis_match_numpy(n):
    rng = np.random.default_rng(100 + n)
    prog = random_program(n, 12 * n, rng)
    st = dense_run(prog, n)                      # n <= 12: shared-memory kernel, else per gate
    ref = np_dense_run(prog, n)
    np.testing.assert_allclose(st.amps, ref, atol=1e-12, rtol=0)
    paulis = random_paulis(n, 24, rng)
    got = st.expectations_pauli(paulis)
    want = np.array([np_expectation(ref, p) for p in paulis])
    np.testing.assert_allclose(got, want, atol=1e-12, rtol=0)
    assert st.expectation_pauli(paulis[0]) == pytest.approx(want[0], abs=1e-12)


def test_per_gate_path_equals_smem_path(rng):
    prog = random_program(9, 80, rng)
    a = dense_run(prog, 9).amps
    st = DenseState(9)
    for instr in prog:
        m = gate_matrix(instr)
        if len(instr.qubits) == 1:
            st.apply_one_qubit(m, instr.qubits[0])
        else:
            st.apply_two_qubit(m, *instr.qubits)
    np.testing.assert_allclose(st.amps, a, atol=1e-13, rtol=0)


def test_batch_states_independent(rng):
    progs = [random_program(6, 40, rng) for _ in range(5)]
    b = DenseBatch(5, 6).run(progs)
    for s, p in enumerate(progs):
        np.testing.assert_allclose(b.amps[s].cpu().numpy(), np_dense_run(p, 6), atol=1e-12, rtol=0)
    paulis = random_paulis(6, 7, rng)
    sidx = np.arange(7) % 5
    got = b.expectations(sidx, paulis)
    want = [np_expectation(np_dense_run(progs[s], 6), p) for s, p in zip(sidx, paulis)]
    np.testing.assert_allclose(got, want, atol=1e-12, rtol=0)


def test_amps_setter_and_amplitude(rng):
    st = DenseState(3)
    v = rng.normal(size=8) + 1j * rng.normal(size=8)
    v /= np.linalg.norm(v)
    st.amps = v
    for bits in ("000", "101", "111"):
        assert st.amplitude(bits) == pytest.approx(v[int(bits, 2)], abs=1e-15)
    with pytest.raises(ValueError):
        st.amplitude("10")


# ---- sampling --------------------------------------------------------------------

@pytest.mark.parametrize("n,seed", [(3, 1), (5, 2), (7, 3)])
def test_sample_counts_identical_to_reference_loop(n, seed):
    prog = random_program(n, 10 * n, np.random.default_rng(seed))
    st = dense_run(prog, n)
    got = st.sample(400, np.random.default_rng(seed + 50))
    want = np_sample(np_dense_run(prog, n), n, 400, np.random.default_rng(seed + 50))
    assert got == want


def test_conditional_prob_zero_matches_numpy(rng):
    n = 5
    prog = random_program(n, 40, rng)
    st = dense_run(prog, n)
    t = np_dense_run(prog, n).reshape((2,) * n)
    for k in range(n):
        for prefix in ("".join(b) for b in itertools.product("01", repeat=k)):
            block = t[tuple(int(b) for b in prefix)]
            p0 = np.sum(np.abs(block[0]) ** 2)
            p1 = np.sum(np.abs(block[1]) ** 2)
            want = p0 / (p0 + p1) if p0 + p1 > 0 else 0.5
            assert st.conditional_prob_zero(prefix, k) == pytest.approx(want, abs=1e-13)


def test_sample_rejects_zero_shots():
    with pytest.raises(ValueError):
        dense_run(bell(), 2).sample(0, np.random.default_rng(0))


# ---- dense <-> MPS cross-checks and the backend switch ---------------------------

def test_run_program_dense_backend_and_execute_counts_match_mps():
    prog = bell() + [I(GateKind.MEASURE, (0,), (), 0), I(GateKind.MEASURE, (1,), (), 1)]
    st = run_program(prog, backend="dense")
    assert isinstance(st, DenseState)
    d = execute(prog, backend="dense", shots=1000, seed=7)
    m = execute(prog, backend="mps", shots=1000, seed=7)
    assert d.counts == m.counts
    assert d.memory_estimate_bytes == 16 * 4 and d.max_bond_seen is None


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_mps_exact_matches_dense(seed):
    rng = np.random.default_rng(seed)
    n = 7
    prog = random_program(n, 60, rng)
    dense = dense_run(prog, n)
    mps = mps_run(prog, n, EXACT)
    keys = ["".join(b) for b in itertools.product("01", repeat=n)]
    mvec = mps.amplitudes(keys)
    assert abs(np.vdot(dense.amps, mvec)) ** 2 == pytest.approx(1.0, abs=1e-10)
    for p in random_paulis(n, 6, rng):
        assert mps.expectation_pauli(p) == pytest.approx(dense.expectation_pauli(p), abs=1e-10)


def test_vqe_sweep_dense_equals_mps():
    n = 4
    body = [I(GateKind.RY, (q,), ("theta",)) for q in range(n)]
    body += [I(GateKind.CNOT, (q, q + 1)) for q in range(n - 1)]
    from paper_1807_07914_b200 import CompositeInstruction
    ans = CompositeInstruction("a", ("theta",), tuple(body))
    ham = PauliHamiltonian(((0.5, "ZZII"), (-1.1, "XIXI"), (0.25, "IYYI"), (0.4, "IIII")))
    d = sweep(ans, ham, -1.0, 1.0, 11, backend="dense")
    m = sweep(ans, ham, -1.0, 1.0, 11, backend="mps", policy=EXACT)
    assert_scaled_close(d.energies, m.energies, 1e-10, "dense vs mps sweep")
    ds = sweep(ans, ham, -1.0, 1.0, 5, backend="dense", shots=300, seed=3)
    ms = sweep(ans, ham, -1.0, 1.0, 5, backend="mps", policy=EXACT, shots=300, seed=3)
    assert ds.energies == ms.energies
