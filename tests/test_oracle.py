"""Pin the CPU oracle (oracle/mps_oracle.py) against golden vectors produced by the
reference itself (oracle/gen_golden.py) and against the dense SVD-free oracle."""

import itertools

import numpy as np
import pytest

from conftest import assert_scaled_close, load_golden, split_lams
from oracle.dense_oracle import dense_amplitude, dense_expectation, dense_run
from oracle.mps_oracle import OracleMps, keep_count, oracle_run
from paper_1807_07914_b200 import workloads as W
from paper_1807_07914_b200.workloads import random_program

RTOL = 1e-10


def _all_bits(n):
    return ["".join(b) for b in itertools.product("01", repeat=n)]


@pytest.mark.parametrize("verbatim", [False, True])
def test_small_cases_match_reference(verbatim):
    g, meta = load_golden("small")
    for i, case in enumerate(meta["cases"]):
        n = case["n"]
        prog = random_program(n, case["gates"], np.random.default_rng(case["seed"]))
        o = oracle_run(prog, n, case["cutoff"], case["max_bond"], case["relative"], verbatim=verbatim)
        bits = _all_bits(n)
        assert_scaled_close([o.amplitude(b) for b in bits], g[f"c{i}_amps"], RTOL, f"case {i}")
        assert_scaled_close([o.expectation(p) for p in case["paulis"]], g[f"c{i}_exps"], RTOL, f"case {i}")
        np.testing.assert_array_equal(o.dims(), g[f"c{i}_dims"])
        for x, y in zip(o.lams, split_lams(g[f"c{i}_lam"], g[f"c{i}_dims"])):
            assert_scaled_close(x, y, RTOL, "lambda")
        assert abs(o.trunc_error_sq - float(g[f"c{i}_trunc_error_sq"])) <= 1e-12
        assert o.max_bond_seen == int(g[f"c{i}_max_bond_seen"])
        assert o.peak_entries == int(g[f"c{i}_peak_entries"])


def test_env_reuse_matches_sweep():
    rng = np.random.default_rng(5)
    n = 8
    o = oracle_run(random_program(n, 60, rng), n, 1e-3, 4)
    paulis = ["".join("IXYZ"[int(c)] for c in rng.integers(0, 4, size=n)) for _ in range(12)]
    paulis += ["I" * n, "Z" + "I" * (n - 1)]
    direct = np.array([o.expectation(p) for p in paulis])
    assert_scaled_close(o.expectations_env(paulis), direct, 1e-12, "env reuse")


def test_exact_mps_matches_dense_oracle():
    rng = np.random.default_rng(11)
    for n in (3, 5, 7):
        prog = random_program(n, 40, rng)
        o = oracle_run(prog, n, 0.0, None)
        psi = dense_run(prog, n)
        bits = _all_bits(n)
        assert_scaled_close([o.amplitude(b) for b in bits], [dense_amplitude(psi, b) for b in bits], 1e-12)
        for q in range(n):
            p = "I" * q + "Z" + "I" * (n - q - 1)
            assert abs(o.expectation(p) - dense_expectation(psi, p)) < 1e-12


def test_keep_count_reference_cases():  # R:tests/test_mps.py:278-283
    s = np.array([1.0, 0.5, 0.3, 1e-9])
    assert keep_count(s, 1e-4, 2) == 2
    assert keep_count(s, 1e-4, None) == 3
    assert keep_count(s, 0.0, None) == 4
    assert keep_count(np.array([1e-20, 1e-30]), 0.5, None, relative=False) == 1


def test_cfg1_matches_reference_golden():
    g, _ = load_golden("cfg1")
    w = W.config1()
    o = oracle_run(w.programs[0], w.n, w.cutoff, w.max_bond)
    assert_scaled_close([o.amplitude(b) for b in w.bitstrings[0]], g["amps"], RTOL, "cfg1 amps")
    assert_scaled_close(o.expectations_env(w.paulis), g["z"], RTOL, "cfg1 <Z>")
    np.testing.assert_array_equal(o.dims(), g["dims"])


def test_cfg2_first_vectors_match_reference_golden():
    g, _ = load_golden("cfg2")
    w = W.config2()
    for v in range(2):
        o = oracle_run(w.programs[v], w.n, w.cutoff, w.max_bond)
        vals = o.expectations_env(w.paulis)
        e = sum(c * x for c, x in zip(w.coeffs.tolist(), vals))
        assert abs(e - g["energies"][v]) <= RTOL * np.max(np.abs(g["energies"]))
        if v == 0:
            assert_scaled_close(vals, g["terms_v0"], RTOL, "cfg2 terms")


def test_cfg4_first_circuits_match_reference_golden():
    g, _ = load_golden("cfg4")
    w = W.config4(circuits=2)
    for c in range(2):
        o = oracle_run(w.programs[c], w.n, w.cutoff, w.max_bond)
        assert abs(o.expectation(w.paulis[0]) - g["zz"][c]) <= RTOL * np.max(np.abs(g["zz"]))
        assert_scaled_close([o.amplitude(b) for b in w.bitstrings[c]], g["amps"][c], RTOL)
        np.testing.assert_array_equal(o.dims(), g["dims"][c])


def test_o2_shim_validation_record():
    import json
    from conftest import GOLDEN
    rec = json.loads((GOLDEN / "o2check.json").read_text())
    assert rec["dims_equal"] and rec["rel_zz"] < 1e-10 and rec["amp_err_of_max"] < 1e-10
