"""vqe.energy / vqe.sweep on the GPU vs the oracle (R:src/mpsqvm/vqe.py:70-125):
analytic energies within 1e-10 of the output scale, sampled (shots) energies
bit-identical because the sampler consumes the reference's uniforms."""

import numpy as np
import pytest

from conftest import assert_scaled_close

pytestmark = pytest.mark.gpu

from oracle.mps_oracle import oracle_run, oracle_sample
from paper_1807_07914_b200 import (CompositeInstruction, GateKind, Instruction, PauliHamiltonian,
                                   TruncationPolicy, bind_parameters, flatten)
from paper_1807_07914_b200.vqe import _basis_rotations, energy, sweep

I = Instruction
N = 6


def ansatz():
    body = [I(GateKind.H, (q,)) for q in range(N)]
    body += [I(GateKind.RY, (q,), ("theta",)) for q in range(N)]
    body += [I(GateKind.CNOT, (q, q + 1)) for q in range(N - 1)]
    inner = CompositeInstruction("mix", ("phi",), tuple(
        [I(GateKind.RZ, (q,), ("theta",)) for q in range(0, N, 2)] +
        [I(GateKind.CZ, (q, q + 1)) for q in range(1, N - 1, 2)] +
        [I(GateKind.RX, (q,), (0.3 * q,)) for q in range(N)]), ("theta",))
    body += [inner, I(GateKind.SWAP, (0, 3)), I(GateKind.MEASURE, (2,), (), 0)]
    return CompositeInstruction("ansatz", ("theta",), tuple(body))


HAM = PauliHamiltonian(((0.5, "ZZIIII"), (-1.2, "XIXIII"), (0.3, "IIIYYI"),
                        (0.7, "IIIIII"), (0.9, "ZIIIIZ")))


def oracle_energy(theta, policy, shots=None, seed=None):
    prog = [i for i in flatten(bind_parameters(ansatz(), [theta])) if i.kind is not GateKind.MEASURE]
    if shots is None:
        o = oracle_run(prog, N, policy.cutoff, policy.max_bond)
        return sum(c * o.expectation(p) for c, p in HAM.terms)
    value = 0.0
    for k, (c, p) in enumerate(HAM.terms):
        if set(p) == {"I"}:
            value += c
            continue
        o = oracle_run(prog + _basis_rotations(p), N, policy.cutoff, policy.max_bond)
        counts = oracle_sample(o, shots, np.random.default_rng([0 if seed is None else seed, k]))
        support = [q for q, ch in enumerate(p) if ch != "I"]
        tot = sum(n if sum(int(b[q]) for q in support) % 2 == 0 else -n for b, n in counts.items())
        value += c * (tot / shots)
    return value


@pytest.mark.parametrize("policy", [TruncationPolicy(), TruncationPolicy(1e-12, 4)])
def test_sweep_analytic_matches_oracle(policy):
    res = sweep(ansatz(), HAM, -1.0, 2.0, 9, policy=policy)
    ref = [oracle_energy(t, policy) for t in res.thetas]
    assert_scaled_close(res.energies, ref, 1e-10, "sweep energies")
    assert res.argmin_theta == res.thetas[int(np.argmin(res.energies))]
    assert res.min_energy == min(res.energies)


def test_energy_with_shots_identical_counts():
    pol = TruncationPolicy()
    for theta in (0.4, -2.1):
        e = energy(ansatz(), theta, HAM, policy=pol, shots=3000, seed=11)
        assert e == oracle_energy(theta, pol, shots=3000, seed=11)


def test_energy_register_check():
    small = PauliHamiltonian(((1.0, "ZZ"),))
    with pytest.raises(ValueError, match="Hamiltonian has 2 qubit"):
        energy(ansatz(), 0.1, small)
