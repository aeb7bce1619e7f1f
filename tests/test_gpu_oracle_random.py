"""Fresh seeded inputs (not in the fixtures) vs the CPU oracle, across bond-size
regimes: single-panel Jacobi (<= 64 columns), block Jacobi + QR preconditioning
(> 64 columns), orientation M / M^H, cutoff / cap / absolute modes, routing."""

import numpy as np
import pytest

from conftest import assert_scaled_close

pytestmark = pytest.mark.gpu

from oracle.mps_oracle import OracleMps, oracle_gate_matrix, oracle_run
from paper_1807_07914_b200 import MatrixGate, MpsBatch, TruncationPolicy, mps_run
from paper_1807_07914_b200.workloads import brick_circuit, haar_unitary, random_bitstrings, random_program

RTOL = 1e-10


def _compare(prog, n, cutoff, chi, relative=True, nbits=32, seed=0):
    st = mps_run(prog, n, TruncationPolicy(cutoff, chi, relative))
    ref = oracle_run(prog, n, cutoff, chi, relative)
    assert [len(v) for v in st.bond_vectors] == ref.dims()
    bits = random_bitstrings(n, nbits, np.random.default_rng(seed))
    assert_scaled_close(st.amplitudes(bits), [ref.amplitude(b) for b in bits], RTOL, "amplitudes")
    paulis = ["I" * q + "Z" + "I" * (n - q - 1) for q in range(n)]
    paulis += ["".join("IXYZ"[int(c)] for c in np.random.default_rng(seed + 1).integers(0, 4, n)) for _ in range(4)]
    assert_scaled_close(st.expectations_pauli(paulis), ref.expectations_env(paulis), RTOL, "expectations")
    for x, y in zip(st.bond_vectors, ref.lams):
        assert_scaled_close(x, y, RTOL, "lambda")
    assert abs(st.trunc_error_sq - ref.trunc_error_sq) <= 1e-10 * max(1.0, ref.trunc_error_sq)
    assert st.max_bond_seen == ref.max_bond_seen and st.peak_entries == ref.peak_entries


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_random_programs_with_routing(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(5, 11))
    _compare(random_program(n, 80, rng), n, [0.0, 1e-3, 1e-8][seed - 1], [None, 6, 16][seed - 1], seed=seed)


def test_absolute_cutoff_mode():
    rng = np.random.default_rng(11)
    _compare(random_program(8, 60, rng), 8, 1e-3, None, relative=False)


@pytest.mark.parametrize("n,depth,chi", [(14, 12, 64), (14, 14, 128)])
def test_block_jacobi_regime(n, depth, chi):
    # chi 64/128 at the centre -> 128/256-column Jacobi with QR preconditioning
    prog = brick_circuit(n, depth, np.random.default_rng(n + depth))
    _compare(prog, n, 1e-12, chi, seed=depth)


def test_haar_two_qubit_gates_and_orientation():
    rng = np.random.default_rng(5)
    n = 12
    prog = []
    for d in range(10):
        for a in range(d % 2, n - 1, 2):
            prog.append(MatrixGate(haar_unitary(rng), (a, a + 1)))
    _compare(prog, n, 1e-12, 48, seed=3)


def test_batched_states_independent():
    rng = np.random.default_rng(21)
    n = 10
    progs = [brick_circuit(n, 8, rng) for _ in range(5)]
    b = MpsBatch(5, n, TruncationPolicy(1e-8, 16))
    b.run(progs)
    paulis = ["Z" + "I" * (n - 2) + "Z", "X" * n]
    for s, p in enumerate(progs):
        ref = oracle_run(p, n, 1e-8, 16)
        vals = b.expectations(np.full(2, s, np.int32), paulis)
        assert_scaled_close(vals, [ref.expectation(x) for x in paulis], RTOL)
        np.testing.assert_array_equal(b.host_dims()[s, 1:n], ref.dims())


def test_load_state_and_single_update_against_oracle():
    """Per-gate drop-in call on an arbitrary (non-canonical) loaded state."""
    rng = np.random.default_rng(8)
    n = 6
    ref = oracle_run(brick_circuit(n, 6, rng), n, 0.0, None)
    st = mps_run([], n, TruncationPolicy(1e-6))
    st._batch.load_state(0, ref.gammas, ref.lams)
    g = haar_unitary(rng)
    st.apply_two_qubit_adjacent(g, 2)
    o = OracleMps(n, 1e-6, None)
    o.gammas = [x.copy() for x in ref.gammas]
    o.lams = [x.copy() for x in ref.lams]
    o.apply_2q(g, 2)
    bits = random_bitstrings(n, 20, rng)
    assert_scaled_close(st.amplitudes(bits), [o.amplitude(b) for b in bits], RTOL)
    assert [len(v) for v in st.bond_vectors] == o.dims()


def test_distributed_energies_nccl_world1():
    import os
    import torch.distributed as dist
    from paper_1807_07914_b200 import workloads as W
    from paper_1807_07914_b200.distributed import vqe_energies
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        w = W.config2(batch=4)
        pol = TruncationPolicy(w.cutoff, w.max_bond)
        e1 = vqe_energies(w.programs, w.n, w.paulis, w.coeffs, pol, mode="by_vector")
        e2 = vqe_energies(w.programs, w.n, w.paulis, w.coeffs, pol, mode="by_term")
    finally:
        dist.destroy_process_group()
    from conftest import load_golden
    g, _ = load_golden("cfg2")
    assert_scaled_close(e1, g["energies"][:4], RTOL)
    assert_scaled_close(e2, g["energies"][:4], RTOL)


def _needs_experimental():
    from paper_1807_07914_b200 import _native
    if not _native.experimental():
        pytest.skip("development variant: libbmps.so built without -DBMPS_EXPERIMENTAL")


def test_tma_staging_path_matches_oracle():
    """The TMA bulk-copy panel staging (tunable tma_staging=1) gives the same results."""
    from paper_1807_07914_b200 import _native
    _needs_experimental()
    with _native.tunables(tma_staging=1):
        prog = brick_circuit(14, 12, np.random.default_rng(99))
        _compare(prog, 14, 1e-12, 64, seed=4)


@pytest.mark.parametrize("mode", [1, 2, 3, 4])
def test_all_jacobi_schedules_match_oracle(mode):
    """persistent / round launches / cluster / dynamic schedules are interchangeable."""
    from paper_1807_07914_b200 import _native
    if mode in (2, 3):
        _needs_experimental()
    with _native.tunables(jacobi_mode=mode):
        prog = brick_circuit(12, 12, np.random.default_rng(7 + mode))
        _compare(prog, 12, 1e-10, 48, seed=mode)


def test_disabled_variants_are_rejected():
    """Without -DBMPS_EXPERIMENTAL the development variants are refused with
    BMPS_E_ARG (surfaced as RuntimeError), never silently replaced; the reserved
    jac_ws field (the removed warp-specialised kernel) is refused in every build."""
    from paper_1807_07914_b200 import _native
    prog = brick_circuit(12, 4, np.random.default_rng(3))
    with _native.tunables(jac_ws=1), pytest.raises(RuntimeError, match="invalid argument"):
        mps_run(prog, 12, TruncationPolicy(1e-10, 64))
    if _native.experimental():
        pytest.skip("experimental build")
    for kw in ({"tma_staging": 1}, {"jacobi_mode": 2}, {"jacobi_mode": 3}):
        with _native.tunables(**kw), pytest.raises(RuntimeError, match="invalid argument"):
            mps_run(prog, 12, TruncationPolicy(1e-10, 64))


@pytest.mark.parametrize("sched", [(0.0, 0, 0.0, 0), (3e-2, 2, 3e-3, 5), (1e-1, 3, 1e-2, 6)])
@pytest.mark.parametrize("chi,cutoff", [(64, 1e-10), (128, 0.0)])
def test_threshold_schedules_match_oracle(sched, chi, cutoff):
    """Threshold Jacobi (thr_a / thr_b: early sweeps defer block pairs whose largest
    relative coupling is under the sweep's threshold): off, the default schedule and a
    coarser one all converge to the oracle's results."""
    from paper_1807_07914_b200 import _native
    ta, sa, tb, sb = sched
    with _native.tunables(thr_a=ta, thr_a_sweeps=sa, thr_b=tb, thr_b_sweeps=sb, thr_auto=0):
        prog = brick_circuit(14, 14, np.random.default_rng(800 + chi))
        _compare(prog, 14, cutoff, chi, seed=chi + sa)


@pytest.mark.parametrize("w2", [16, 64])
@pytest.mark.parametrize("chi,cutoff", [(64, 1e-10), (128, 0.0)])
def test_other_panel_widths_match_oracle(w2, chi, cutoff):
    """block_w2 = 16 / 64: visits of 16- and 64-column panels (2 and 8 column groups in
    the batched inner sweep, deferred Q update on 7 / 4 spare warps) instead of 32."""
    from paper_1807_07914_b200 import _native
    with _native.tunables(block_w2=w2):
        prog = brick_circuit(14, 14, np.random.default_rng(700 + chi + w2))
        _compare(prog, 14, cutoff, chi, seed=chi + w2)


@pytest.mark.parametrize("dq", [0, 1])
@pytest.mark.parametrize("chi,cutoff", [(64, 1e-12), (128, 1e-10), (128, 0.0)])
def test_double_qr_preconditioning_matches_oracle(dq, chi, cutoff):
    """Single vs double Householder-QR preconditioning (tunable double_qr)."""
    from paper_1807_07914_b200 import _native
    with _native.tunables(double_qr=dq):
        prog = brick_circuit(14, 14, np.random.default_rng(chi + dq))
        _compare(prog, 14, cutoff, chi, seed=chi)


@pytest.mark.parametrize("small", [1, 0])
@pytest.mark.parametrize("chi,cutoff,n", [(64, 1e-10, 14), (128, 0.0, 14), (40, 1e-12, 13)])
def test_short_qr_panel_kernel_matches_oracle(small, chi, cutoff, n):
    """qr_small: QR panels of <= 128 rows on the 128-thread short-panel kernel (forced on
    for these small batches; auto only takes it when the batch exceeds the SM count) or
    on the 512-thread kernel (0). chi = 40 gives ragged panels (80 columns: 32 + 32 + 16)."""
    from paper_1807_07914_b200 import _native
    with _native.tunables(qr_small=small):
        prog = brick_circuit(n, 14, np.random.default_rng(600 + chi))
        _compare(prog, n, cutoff, chi, seed=chi + 1)


@pytest.mark.parametrize("csize", [0, 2, 4])
@pytest.mark.parametrize("chi,cutoff", [(64, 1e-10), (128, 0.0)])
def test_row_split_cluster_jacobi_matches_oracle(csize, chi, cutoff):
    """jac_cluster: each visit's panel rows split over a 2- or 4-CTA cluster (partial
    Grams summed through distributed shared memory), or off (0)."""
    from paper_1807_07914_b200 import _native
    with _native.tunables(jac_cluster=csize):
        prog = brick_circuit(14, 14, np.random.default_rng(900 + chi + csize))
        _compare(prog, 14, cutoff, chi, seed=chi + csize)


def _theta(gammas, lams, q):
    """Gauge-invariant two-site tensor lam_{q-1} G_q lam_q G_{q+1} lam_{q+1} (mps.py:105-109)."""
    n = len(gammas)
    lam_l = lams[q - 1] if q > 0 else np.ones(1)
    lam_r = lams[q + 1] if q + 1 < n - 1 else np.ones(1)
    return np.einsum("l,lsm,m,mtr,r->lstr", lam_l, gammas[q], lams[q], gammas[q + 1], lam_r, optimize=True)


@pytest.mark.parametrize("qr_cluster", [1, 0])
def test_chi256_updates_on_cfg3_steady_state_match_oracle(qr_cluster):
    """The bench's unit of work at full size: chi = 256 CNOT updates (512 x 512 theta,
    keep 256 of 512) on a GPU-evolved cfg3 state (50 qubits, 25 layers), against the
    oracle applied to the same tensors: new bond vector and the two-site tensor.
    The 512-row QR panels run on 2-CTA row-split clusters (qr_cluster=1, default) or
    one CTA streaming from L2 (0)."""
    from paper_1807_07914_b200 import _native
    with _native.tunables(qr_cluster=qr_cluster):
        _chi256_steady_state_case()


def _chi256_steady_state_case():
    import bench
    from paper_1807_07914_b200.ir import GateKind, Instruction
    st = mps_run(bench.prefix_program(1003, 25), bench.N_QUBITS, TruncationPolicy(bench.CUTOFF, bench.CHI))
    gam, lam = st.site_tensors, st.bond_vectors
    sites = [q for q in range(10, 38, 9) if len(lam[q - 1]) == len(lam[q]) == len(lam[q + 1]) == 256]
    assert sites, "no all-256 site pair in the steady state"
    o = OracleMps(bench.N_QUBITS, bench.CUTOFF, bench.CHI)
    o.gammas = [g.copy() for g in gam]
    o.lams = [v.copy() for v in lam]
    cnot = oracle_gate_matrix(Instruction(GateKind.CNOT, (0, 1)))
    err0 = st.trunc_error_sq
    for q in sites:
        st.apply_two_qubit_adjacent(cnot, q)
        o.apply_2q(cnot, q)
    gam2, lam2 = st.site_tensors, st.bond_vectors
    for q in sites:
        assert len(lam2[q]) == len(o.lams[q]) == 256
        assert_scaled_close(lam2[q], o.lams[q], RTOL, f"lambda bond {q}")
        assert_scaled_close(_theta(gam2, lam2, q).ravel(), _theta(o.gammas, o.lams, q).ravel(), RTOL,
                            f"theta sites {q},{q + 1}")
    d_err = st.trunc_error_sq - err0
    assert abs(d_err - o.trunc_error_sq) <= 1e-10 * max(1.0, o.trunc_error_sq)


@pytest.mark.parametrize("count", [1, 3, 7, 29])
def test_batched_amplitudes_mixed_states(count):
    """bmps_amplitudes groups consecutive same-state bitstrings per CTA; interleaved
    states (mixed groups) and ragged counts must give the oracle's amplitudes and be
    bit-identical to one call per bitstring."""
    n, S = 8, 3
    rng = np.random.default_rng(40 + count)
    progs = [brick_circuit(n, 6, np.random.default_rng(100 + s)) for s in range(S)]
    b = MpsBatch(S, n, TruncationPolicy(0.0, 8))
    b.run(progs)
    b.check_status()
    refs = [oracle_run(p, n, 0.0, 8, True) for p in progs]
    states = rng.integers(0, S, count).astype(np.int32)
    states[: min(count, 2)] = 0   # at least one same-state run when count > 1
    bits = random_bitstrings(n, count, rng)
    got = b.amplitudes(states, bits)
    assert_scaled_close(got, [refs[s].amplitude(x) for s, x in zip(states, bits)], RTOL, "amplitudes")
    one = np.array([b.amplitudes(states[i:i + 1], bits[i:i + 1])[0] for i in range(count)])
    assert np.array_equal(got, one)
