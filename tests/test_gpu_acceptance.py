"""The reference's acceptance criteria for the MPS hot path (R:tests/test_acceptance.py,
SPEC criteria 1-5; criterion 6 lives in test_gpu_dense.py::test_vqe_sweep_dense_equals_mps)
and the two test_mps.py cases the survey lists beside them, re-targeted at the drop-in
API on the GPU. The SVD-free cross-check is the GPU dense backend, as the reference uses
its dense oracle; tolerances are the reference's own."""

import itertools
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_1807_07914_b200 import (GateKind, Instruction, MpsState, TruncationPolicy, dense_run,
                                   gate_matrix, mps_run, simulate_batch)
from paper_1807_07914_b200.workloads import random_program, round_circuit

EXACT = TruncationPolicy(cutoff=0.0)


def _statevector(state):
    """R:tests/conftest.py:36-40 (through the batched amplitude call)."""
    return state.amplitudes(["".join(b) for b in itertools.product("01", repeat=state.n)])


def test_round_circuit_matches_the_reference_generator_structure():
    # R:tests/test_bench.py:29-47
    prog = round_circuit(6, 2, 3)
    assert [i.kind for i in prog[:6]] == [GateKind.H] * 6
    cnots = [i.qubits for i in prog if i.kind is GateKind.CNOT]
    assert cnots == [(0, 1), (2, 3), (4, 5), (1, 2), (3, 4)]
    assert round_circuit(6, 2, 3)[6].params == prog[6].params
    with pytest.raises(ValueError):
        round_circuit(1, 2, 0)
    with pytest.raises(ValueError):
        round_circuit(4, 0, 0)


def test_criterion_1_oracle_equivalence():
    """R:tests/test_acceptance.py:76-101: 200 random circuits, n in [2, 8], <= 30 gates,
    cutoff 0, cap 2^ceil(n/2): fidelity against the dense backend and every <Z_q>."""
    rng = np.random.default_rng(20240)
    worst_f, worst_z = 1.0, 0.0
    for _ in range(200):
        n = int(rng.integers(2, 9))
        program = random_program(n, int(rng.integers(5, 31)), rng)
        mps = mps_run(program, n, TruncationPolicy(cutoff=0.0, max_bond=2 ** ((n + 1) // 2)))
        dense = dense_run(program, n)
        fidelity = abs(np.vdot(dense.amps, _statevector(mps))) ** 2
        worst_f = min(worst_f, fidelity)
        assert fidelity >= 1 - 1e-10
        paulis = ["I" * q + "Z" + "I" * (n - q - 1) for q in range(n)]
        gap = np.abs(mps.expectations_pauli(paulis) - np.array([dense.expectation_pauli(p) for p in paulis]))
        worst_z = max(worst_z, float(gap.max()))
        assert gap.max() < 1e-9
    print(f"criterion 1: worst fidelity {worst_f:.3e}, worst <Z> gap {worst_z:.3e}")


def test_criterion_2_two_round_bond_law():
    """R:tests/test_acceptance.py:104-115: chi = 4 after two rounds for n = 5..40 and ten
    seeds each -- the ten seeds of an n as one batch -- and the per-gate storage law
    (memory <= 16 (2 n chi^2 + (n - 1) chi) after every gate) through the per-gate API."""
    for n in range(5, 45, 5):
        batch = simulate_batch([round_circuit(n, 2, seed) for seed in range(10)], n, EXACT)
        assert [int(x) for x in batch.stats()["max_bond_seen"]] == [4] * 10
    n = 20
    state = MpsState(n, EXACT)
    for instr in round_circuit(n, 2, 0):
        if len(instr.qubits) == 1:
            state.apply_one_qubit(gate_matrix(instr), instr.qubits[0])
        else:
            state.apply_two_qubit_routed(gate_matrix(instr), *instr.qubits)
        chi = state.max_bond_seen
        assert state.memory_estimate_bytes() <= 16 * (2 * n * chi ** 2 + (n - 1) * chi)
    assert state.max_bond_seen == 4


def test_criterion_3_saturation_law():
    """R:tests/test_acceptance.py:118-127: chi = 2^(n/2) after 2n rounds at cutoff 0."""
    for n, expected in ((6, 8), (8, 16), (10, 32)):
        assert mps_run(round_circuit(n, 2 * n, 0), n, EXACT).max_bond_seen == expected


def test_criterion_4_storage_law_linearity():
    """R:tests/test_acceptance.py:130-149: at two rounds the memory grows linearly in n."""
    ns = list(range(5, 45, 5))
    means = []
    for n in ns:
        batch = simulate_batch([round_circuit(n, 2, seed) for seed in range(10)], n, EXACT)
        means.append(float(np.mean(16 * batch.stats()["peak_entries"])))   # memory_estimate_bytes
    fit = np.polyfit(ns, means, 1)
    res = np.sum((np.array(means) - np.polyval(fit, ns)) ** 2)
    tot = np.sum((np.array(means) - np.mean(means)) ** 2)
    assert 1 - res / tot > 0.999


def test_criterion_5_large_shallow_run():
    """R:tests/test_acceptance.py:152-160: 85 qubits, two rounds, cutoff 1e-4: under 10 s
    and under 1e5 bytes."""
    mps_run(round_circuit(8, 2, 1), 8, TruncationPolicy(cutoff=1e-4)).synchronize()   # warm-up
    t0 = time.perf_counter()
    state = mps_run(round_circuit(85, 2, 0), 85, TruncationPolicy(cutoff=1e-4))
    mem = state.memory_estimate_bytes()
    assert time.perf_counter() - t0 < 10
    assert mem < 10 ** 5


def test_routing_neutral_ordering_exhaustive():
    """R:tests/test_mps.py:138-152: all 64 amplitudes after routed CNOT (5, 1) and CZ (0, 4)."""
    rng = np.random.default_rng(2024)
    program = random_program(6, 12, rng, two_qubit_prob=0.0)
    program += [Instruction(GateKind.CNOT, (5, 1)), Instruction(GateKind.CZ, (0, 4))]
    np.testing.assert_allclose(_statevector(mps_run(program, 6, EXACT)), dense_run(program, 6).amps,
                               rtol=0, atol=1e-10)


def test_truncation_error_bounds_infidelity():
    """R:tests/test_mps.py:246-261: infidelity <= 4 trunc_error_sq at cutoff 0.05."""
    rng = np.random.default_rng(2024)
    checked = 0
    for _ in range(20):
        n = int(rng.integers(4, 9))
        program = random_program(n, 30, rng)
        state = mps_run(program, n, TruncationPolicy(cutoff=0.05))
        if state.trunc_error_sq < 1e-12:
            continue
        vec = _statevector(state)
        infidelity = 1 - abs(np.vdot(dense_run(program, n).amps, vec)) ** 2 / np.vdot(vec, vec).real
        assert infidelity <= 4 * state.trunc_error_sq + 1e-12
        checked += 1
    assert checked >= 3
