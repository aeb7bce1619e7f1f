"""GPU sequential sampling vs the reference semantics (R:tests/test_mps.py:189-218)
and exact count parity with the oracle port on seeded generators."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle.dense_oracle import dense_run
from oracle.mps_oracle import oracle_run, oracle_sample
from paper_1807_07914_b200 import GateKind, Instruction, TruncationPolicy, execute, mps_run
from paper_1807_07914_b200.workloads import brick_circuit, random_program

EXACT = TruncationPolicy(cutoff=0.0)


def bell():
    return [Instruction(GateKind.H, (0,)), Instruction(GateKind.CNOT, (0, 1))]


def test_computational_basis_state():
    st = mps_run([Instruction(GateKind.X, (0,)), Instruction(GateKind.X, (1,))], 2)
    assert st.sample(100, np.random.default_rng(0)) == {"11": 100}


def test_bell_within_5_sigma():
    counts = mps_run(bell(), 2, EXACT).sample(100_000, np.random.default_rng(1))
    assert set(counts) <= {"00", "11"}
    assert abs(counts["00"] - 50_000) < 5 * np.sqrt(100_000 * 0.25)


def test_deterministic_given_seed():
    st = mps_run(bell(), 2, EXACT)
    assert st.sample(500, np.random.default_rng(9)) == st.sample(500, np.random.default_rng(9))


def test_tvd_vs_dense_distribution(rng):
    prog = random_program(4, 20, rng)
    counts = mps_run(prog, 4, EXACT).sample(100_000, np.random.default_rng(3))
    psi = dense_run(prog, 4)
    probs = {format(i, "04b"): abs(a) ** 2 for i, a in enumerate(psi)}
    tvd = 0.5 * sum(abs(counts.get(b, 0) / 100_000 - p) for b, p in probs.items())
    assert tvd < 0.02


@pytest.mark.parametrize("n,depth,cutoff,chi", [(8, 6, 0.0, None), (12, 8, 1e-4, 8), (16, 10, 1e-10, 32)])
def test_counts_identical_to_oracle(n, depth, cutoff, chi):
    prog = brick_circuit(n, depth, np.random.default_rng(n * 100 + depth))
    gpu = mps_run(prog, n, TruncationPolicy(cutoff, chi)).sample(2000, np.random.default_rng(77))
    ref = oracle_sample(oracle_run(prog, n, cutoff, chi), 2000, np.random.default_rng(77))
    assert gpu == ref


def test_execute_marginalises_measured_qubits():
    prog = bell() + [Instruction(GateKind.MEASURE, (1,)), Instruction(GateKind.MEASURE, (0,))]
    rec = execute(prog, 2, policy=EXACT, shots=1000, seed=5)
    assert set(rec.counts) <= {"00", "11"} and sum(rec.counts.values()) == 1000
    assert rec.max_bond_seen == 2 and rec.memory_estimate_bytes == 16 * 8
