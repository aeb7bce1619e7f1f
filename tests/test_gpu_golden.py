"""GPU parity against golden vectors produced by the reference itself (oracle/gen_golden.py).

Gauge-invariant quantities only: amplitudes, Pauli expectations,
Schmidt spectra, bond dims (exact), trunc_error_sq, stats (exact). Tolerance:
|delta| <= 1e-10 * max|ref| over each output set.
"""

import numpy as np
import pytest

from conftest import assert_scaled_close, load_golden, split_lams

pytestmark = pytest.mark.gpu

from paper_1807_07914_b200 import MpsBatch, TruncationPolicy, compile_batch, mps_run
from paper_1807_07914_b200 import workloads as W
from paper_1807_07914_b200.workloads import random_program

RTOL = 1e-10


def _check_state_summary(batch, s, g, prefix, lam_rtol=RTOL):
    dims = batch.host_dims()[s][1:batch.n]
    np.testing.assert_array_equal(dims, g[prefix + "dims"], err_msg="bond dims")
    ref_l = split_lams(g[prefix + "lam"], g[prefix + "dims"])
    got_l = batch.bond_vectors(s)
    for b, (x, y) in enumerate(zip(got_l, ref_l)):
        assert_scaled_close(x, y, lam_rtol, f"lambda bond {b}")
    st = batch.stats()
    te_ref = float(g[prefix + "trunc_error_sq"])
    assert abs(st["trunc_error_sq"][s] - te_ref) <= 1e-10 * max(1.0, te_ref)
    assert int(st["max_bond_seen"][s]) == int(g[prefix + "max_bond_seen"])
    assert int(st["peak_entries"][s]) == int(g[prefix + "peak_entries"])


def test_small_programs():
    g, meta = load_golden("small")
    for i, case in enumerate(meta["cases"]):
        n = case["n"]
        pol = TruncationPolicy(case["cutoff"], case["max_bond"], case["relative"])
        prog = random_program(n, case["gates"], np.random.default_rng(case["seed"]))
        st = mps_run(prog, n, pol)
        bits = ["".join(b) for b in np.array(np.meshgrid(*[["0", "1"]] * n, indexing="ij")).reshape(n, -1).T]
        assert_scaled_close(st.amplitudes(bits), g[f"c{i}_amps"], RTOL, f"case {i} amplitudes")
        assert_scaled_close(st.expectations_pauli(case["paulis"]), g[f"c{i}_exps"], RTOL, f"case {i} expectations")
        assert abs(st.norm_sq() - float(g[f"c{i}_norm"])) <= 1e-10
        _check_state_summary(st._batch, 0, g, f"c{i}_")


def test_cfg1():
    g, _ = load_golden("cfg1")
    w = W.config1()
    st = mps_run(w.programs[0], w.n, TruncationPolicy(w.cutoff, w.max_bond))
    assert_scaled_close(st.amplitudes(w.bitstrings[0]), g["amps"], RTOL, "cfg1 amplitudes")
    assert_scaled_close(st.expectations_pauli(w.paulis), g["z"], RTOL, "cfg1 <Z>")
    _check_state_summary(st._batch, 0, g, "")


def test_cfg2_energies():
    from paper_1807_07914_b200.vqe import energies
    g, _ = load_golden("cfg2")
    w = W.config2()
    e = energies(w.programs, w.n, w.paulis, w.coeffs, TruncationPolicy(w.cutoff, w.max_bond))
    assert_scaled_close(e, g["energies"], RTOL, "cfg2 energies")


def test_cfg3():
    g, _ = load_golden("cfg3")
    w = W.config3()
    b = MpsBatch(1, w.n, TruncationPolicy(w.cutoff, w.max_bond))
    b.run(w.programs)
    z = b.expectations(np.zeros(w.n, np.int32), w.paulis)
    assert_scaled_close(z, g["z"], RTOL, "cfg3 <Z>")
    assert abs(b.expectations([0], ["I" * w.n])[0] - float(g["norm"])) <= 1e-10 * float(g["norm"])
    assert_scaled_close(b.bond_truncation(0), g["bond_err"], RTOL, "cfg3 per-bond truncation")
    _check_state_summary(b, 0, g, "")


def test_cfg4_sample():
    g, meta = load_golden("cfg4")
    cnt = meta["circuits"]
    w = W.config4(circuits=cnt)
    b = MpsBatch(cnt, w.n, TruncationPolicy(w.cutoff, w.max_bond))
    b.run(w.programs)
    zz = b.expectations(np.arange(cnt, dtype=np.int32), w.paulis * cnt)
    assert_scaled_close(zz, g["zz"], RTOL, "cfg4 <Z0 Z31>")
    for c in range(cnt):
        amps = b.amplitudes(np.full(16, c, np.int32), w.bitstrings[c])
        assert_scaled_close(amps, g["amps"][c], RTOL, f"cfg4 amplitudes circuit {c}")
    np.testing.assert_array_equal(b.host_dims()[:, 1:w.n], g["dims"])
    st = b.stats()
    np.testing.assert_allclose(st["trunc_error_sq"], g["trunc_error_sq"], rtol=1e-10)
    np.testing.assert_array_equal(st["max_bond_seen"], g["max_bond_seen"])


def test_cfg5():
    g, _ = load_golden("cfg5")
    w = W.config5()
    b = MpsBatch(1, w.n, TruncationPolicy(w.cutoff, w.max_bond))
    b.run(w.programs)
    np.testing.assert_array_equal(b.host_dims()[0, 1:w.n], g["dims"])
    vals = b.expectations(np.zeros(2 * w.n, np.int32), w.paulis)
    assert_scaled_close(vals[: w.n], g["x"], RTOL, "cfg5 <X>")
    assert_scaled_close(vals[w.n:], g["z"], RTOL, "cfg5 <Z>")
    assert_scaled_close(b.bond_truncation(0), g["bond_err"], 1e-8, "cfg5 per-bond truncation")
    st = b.stats()
    assert abs(st["trunc_error_sq"][0] - float(g["trunc_error_sq"])) <= 1e-8 * float(g["trunc_error_sq"])
    assert int(st["max_bond_seen"][0]) == int(g["max_bond_seen"])
    lam = b.bond_vectors(0)
    for k, v in enumerate(lam):
        head = g["lam_head"][k][: min(8, len(v))]
        assert_scaled_close(v[: len(head)], head, RTOL, f"cfg5 lambda head bond {k}")


@pytest.mark.parametrize("param,value", [("jac_cluster", 4.0), ("jac_cluster", 2.0), ("jac_ws", 1.0)])
@pytest.mark.parametrize("cfg", ["cfg3", "cfg5"])
def test_golden_under_jacobi_variants(cfg, param, value):
    """The config-scale goldens (cfg3: chi 256, cfg5: chi 1024) through the row-split
    cluster kernel forced on every layer and through the warp-specialised kernel."""
    from paper_1807_07914_b200 import _native
    lib = _native.load()
    assert lib.bmps_set_param(param.encode(), value) == 0
    try:
        (test_cfg3 if cfg == "cfg3" else test_cfg5)()
    finally:
        lib.bmps_set_param(param.encode(), float(_native.DEFAULT_PARAMS[param]))
