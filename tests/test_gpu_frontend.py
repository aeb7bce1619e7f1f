"""Kernel text -> reference ``parse`` (offline, oracle/gen_frontend.py) -> this
package's ``bind_parameters`` / ``flatten`` -> GPU executor, against the
reference's own answers (R:src/mpsqvm/parser.py:242,
ir.py:150-184, vqe.py:87-89, vqe.py:100-125)."""

import numpy as np
import pytest

from conftest import assert_scaled_close
from frontend_fixture import hamiltonian, load_frontend, tree_from_json

pytestmark = pytest.mark.gpu

from paper_1807_07914_b200 import IrError, TruncationPolicy, bind_parameters, flatten, mps_run
from paper_1807_07914_b200.vqe import parameter_energies, sweep

RTOL = 1e-10


@pytest.mark.parametrize("pi", [0, 1])
def test_multi_parameter_energies_match_reference(pi):
    fx = load_frontend()
    m = fx["multi"][pi]
    ansatz = tree_from_json(fx["kernels"]["ansatz"])
    pol = TruncationPolicy(m["cutoff"], m["max_bond"])
    e = parameter_energies(ansatz, fx["vectors"], hamiltonian(fx), policy=pol)
    assert_scaled_close(e, m["energies"], RTOL, "multi-parameter energies")
    for v, vec in enumerate(fx["vectors"]):
        prog = [i for i in flatten(bind_parameters(ansatz, vec)) if i.kind.value != "MEASURE"]
        st = mps_run(prog, fx["n"], pol)
        ref = np.array([complex(*a) for a in m["amps"][v]])
        assert_scaled_close(st.amplitudes(fx["bits"]), ref, RTOL, f"amplitudes vector {v}")
        assert [len(x) for x in st.bond_vectors] == m["dims"][v]


def test_multi_parameter_rejects_wrong_arity():
    fx = load_frontend()
    ansatz = tree_from_json(fx["kernels"]["ansatz"])
    with pytest.raises(IrError, match="takes 4 parameter"):
        parameter_energies(ansatz, [[0.1, 0.2]], hamiltonian(fx))


@pytest.mark.parametrize("pi", [0, 1])
def test_single_parameter_sweep_matches_reference_driver(pi):
    fx = load_frontend()
    s = fx["sweeps"][pi]
    res = sweep(tree_from_json(fx["kernels"]["single"]), hamiltonian(fx), -1.0, 2.0, 7, "mps",
                TruncationPolicy(s["cutoff"], s["max_bond"]))
    np.testing.assert_array_equal(res.thetas, s["thetas"])
    assert_scaled_close(res.energies, s["energies"], RTOL, "sweep energies")
    assert res.argmin_theta == s["argmin_theta"]
    assert abs(res.min_energy - s["min_energy"]) <= RTOL * max(1.0, abs(s["min_energy"]))


def test_sweep_keeps_reference_single_parameter_contract():
    fx = load_frontend()
    with pytest.raises(ValueError, match="exactly one formal parameter"):
        sweep(tree_from_json(fx["kernels"]["ansatz"]), hamiltonian(fx), count=3)
