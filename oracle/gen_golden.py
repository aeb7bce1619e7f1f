"""Generate golden fixtures from the REFERENCE itself -- TEST INFRASTRUCTURE ONLY.

Runs the unmodified reference package (``/root/reference/pkg/src/mpsqvm``,
imported read-only in the build container; it does not exist on the GPU box)
on the seeded workloads of ``paper_1807_07914_b200.workloads`` and writes
``tests/golden/<case>.npz``. Modes, following SURVEY.md §8(c):

* O1 "verbatim": the reference as shipped (``mps_run`` semantics, its einsums);
* O2 "shim": the same reference code with ``mpsqvm.mps.np`` replaced by a
  namespace whose ``einsum`` forces ``optimize=True`` (contraction order only;
  SVD, truncation, pseudo-inverse and renormalisation code paths unchanged);
* O2+: many single-site expectations via cached environments, evaluated by
  ``oracle.mps_oracle.OracleMps.expectations_env`` on the reference's final
  Gamma/lambda (the ``mps.py:196-204`` sum reassociated).

Usage: ``python -m oracle.gen_golden small cfg1 cfg2 cfg4 o2check cfg3 cfg5``.
"""

from __future__ import annotations

import json
import os
import sys
import time
import types
from pathlib import Path

import numpy as np

REF_SRC = "/root/reference/pkg/src"
ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))
sys.dont_write_bytecode = True


def _ref():
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import mpsqvm  # noqa: F401  (reference package, read-only)
    import mpsqvm.mps as ref_mps
    return mpsqvm, ref_mps


class _NpShim(types.ModuleType):
    """numpy namespace whose einsum always uses optimize=True (the O2 shim)."""

    def __getattr__(self, name):
        return getattr(np, name)


class _SvdRecorder(types.ModuleType):
    """``np.linalg`` whose ``svd`` also keeps the raw singular values it returns
    (the numbers ``keep_count`` decides on, ``mps.py:116-120``); the call itself is
    numpy's, so results are bit-identical to the unpatched reference."""

    def __init__(self, name):
        super().__init__(name)
        self.spectra = []

    def __getattr__(self, name):
        return getattr(np.linalg, name)

    def svd(self, *a, **k):
        out = np.linalg.svd(*a, **k)
        self.spectra.append(np.array(out[1]))
        return out


def set_shim(on: bool, record: bool = False):
    """O2 shim on/off; with ``record`` the reference's SVD spectra are captured
    (returns the recorder)."""
    _, ref_mps = _ref()
    rec = None
    if on or record:
        shim = _NpShim("numpy_o2")
        if on:
            shim.einsum = lambda *a, **k: np.einsum(*a, **{**k, "optimize": True})
        if record:
            rec = _SvdRecorder("numpy_linalg_rec")
            shim.linalg = rec
        ref_mps.np = shim
    else:
        ref_mps.np = np
    return rec


def decision_margins(spectra, cutoff, max_bond, relative=True):
    """Per update: the keep count of ``TruncationPolicy.keep_count`` (``mps.py:43-49``),
    the distance of the nearest singular value that can move it from the cutoff
    threshold, ``min_{k < min(p, max_bond)} |sigma_k - thr| / sigma_0`` (inf when
    cutoff is 0), and the spectral gap at the truncation boundary
    ``(sigma_{keep-1} - sigma_keep) / sigma_0`` (inf when nothing is discarded)."""
    keep, margin, gap = [], [], []
    for s in spectra:
        p = len(s)
        s0 = float(s[0]) if p else 0.0
        if cutoff > 0:
            thr = cutoff * (s0 if relative else 1.0)
            k = int(np.sum(s >= thr))
        else:
            thr, k = None, p
        k = max(k, 1)
        if max_bond is not None:
            k = min(k, max_bond)
        K = p if max_bond is None else min(p, max_bond)
        if thr is None or s0 == 0.0:
            m = np.inf
        else:
            m = float(np.min(np.abs(s[:K] - thr))) / s0
        g = float(s[k - 1] - s[k]) / s0 if k < p and s0 > 0 else np.inf
        keep.append(k)
        margin.append(m)
        gap.append(g)
    return np.array(keep, np.int64), np.array(margin), np.array(gap)


def ref_matrix(op):
    """Gate matrix through the reference's own ``gate_matrix`` (pins conventions)."""
    mpsqvm, _ = _ref()
    from mpsqvm.gates import gate_matrix
    if getattr(op, "matrix", None) is not None:
        return np.asarray(op.matrix, dtype=complex)
    rop = mpsqvm.Instruction(mpsqvm.GateKind(op.kind.value), tuple(op.qubits), tuple(op.params))
    return gate_matrix(rop)


def ref_evolve(program, n, cutoff, max_bond, relative=True, per_bond=False):
    """``backends.mps_run`` loop on the reference MpsState (explicit matrices allowed)."""
    mpsqvm, ref_mps = _ref()
    state = ref_mps.MpsState(n, ref_mps.TruncationPolicy(cutoff, max_bond, relative))
    bond_err = np.zeros(max(n - 1, 0))
    if per_bond:
        orig = state.apply_two_qubit_adjacent

        def wrapped(gate, q):
            before = state.trunc_error_sq
            orig(gate, q)
            bond_err[q] += state.trunc_error_sq - before
        state.apply_two_qubit_adjacent = wrapped
    for op in program:
        kind = getattr(op, "kind", None)
        if kind is not None and kind.value == "MEASURE":
            continue
        g = ref_matrix(op)
        if len(op.qubits) == 1:
            state.apply_one_qubit(g, op.qubits[0])
        else:
            state.apply_two_qubit_routed(g, op.qubits[0], op.qubits[1])
    return state, bond_err


def state_summary(state) -> dict:
    dims = np.array([len(v) for v in state.bond_vectors], dtype=np.int64)
    lam = np.concatenate(state.bond_vectors) if state.bond_vectors else np.zeros(0)
    return {
        "dims": dims, "lam": lam, "trunc_error_sq": np.float64(state.trunc_error_sq),
        "max_bond_seen": np.int64(state.max_bond_seen), "peak_entries": np.int64(state.peak_entries),
    }


def to_oracle(state):
    from oracle.mps_oracle import OracleMps
    o = OracleMps(state.n)
    o.gammas = [np.array(t) for t in state.site_tensors]
    o.lams = [np.array(v) for v in state.bond_vectors]
    return o


def save(name: str, meta: dict, **arrays) -> None:
    GOLDEN.mkdir(parents=True, exist_ok=True)
    np.savez_compressed(GOLDEN / f"{name}.npz", meta=json.dumps(meta), **arrays)
    print(f"wrote {name}.npz ({(GOLDEN / f'{name}.npz').stat().st_size} B)", flush=True)


SMALL_POLICIES = [
    (0.0, None, True), (1e-4, None, True), (0.05, None, True),
    (1e-4, 2, True), (0.0, 4, True), (1e-3, None, False),
]


def gen_small() -> None:
    """Small random programs (n=2..8, non-adjacent pairs) under several policies."""
    from paper_1807_07914_b200.workloads import random_program
    set_shim(False)
    master = np.random.default_rng(20241020)
    cases = []
    out = {}
    for i in range(48):
        n = int(master.integers(2, 9))
        gates = int(master.integers(10, 41))
        seed = int(master.integers(1 << 31))
        cutoff, max_bond, relative = SMALL_POLICIES[i % len(SMALL_POLICIES)]
        prog = random_program(n, gates, np.random.default_rng(seed))
        state, _ = ref_evolve(prog, n, cutoff, max_bond, relative)
        bits = ["".join(b) for b in np.array(np.meshgrid(*[["0", "1"]] * n, indexing="ij")).reshape(n, -1).T]
        amps = np.array([state.amplitude(b) for b in bits])
        prng = np.random.default_rng(seed + 1)
        paulis = ["I" * q + "Z" + "I" * (n - q - 1) for q in range(n)]
        paulis += ["".join("IXYZ"[int(c)] for c in prng.integers(0, 4, size=n)) for _ in range(4)]
        exps = np.array([state.expectation_pauli(p) for p in paulis])
        summ = state_summary(state)
        cases.append({"n": n, "gates": gates, "seed": seed, "cutoff": cutoff,
                      "max_bond": max_bond, "relative": relative, "paulis": paulis})
        out[f"c{i}_amps"] = amps
        out[f"c{i}_exps"] = exps
        out[f"c{i}_norm"] = np.float64(state.norm_sq())
        for k, v in summ.items():
            out[f"c{i}_{k}"] = v
    save("small", {"cases": cases}, **out)


def gen_cfg1() -> None:
    from paper_1807_07914_b200.workloads import config1
    w = config1()
    rec = set_shim(False, record=True)
    t0 = time.perf_counter()
    state, _ = ref_evolve(w.programs[0], w.n, w.cutoff, w.max_bond)
    t_ev = time.perf_counter() - t0
    keep, margin, gap = decision_margins(rec.spectra, w.cutoff, w.max_bond)
    amps = np.array([state.amplitude(b) for b in w.bitstrings[0]])
    set_shim(True)
    t0 = time.perf_counter()
    z = np.array([state.expectation_pauli(p) for p in w.paulis])
    t_q = time.perf_counter() - t0
    set_shim(False)
    save("cfg1", {"mode": "O1 evolution + amplitudes; O2 shim for <Z>", "evolve_s": t_ev,
                  "query_s": t_q, "seed": w.meta["seed"]},
         amps=amps, z=z, upd_keep=keep, upd_margin=margin, upd_gap=gap, **state_summary(state))


def gen_cfg2() -> None:
    from paper_1807_07914_b200.workloads import config2
    w = config2()
    set_shim(True)
    energies = np.empty(len(w.programs))
    term0 = None
    t0 = time.perf_counter()
    dims = []
    for v, prog in enumerate(w.programs):
        state, _ = ref_evolve(prog, w.n, w.cutoff, w.max_bond)
        vals = [state.expectation_pauli(p) for p in w.paulis]
        energies[v] = sum(c * e for c, e in zip(w.coeffs.tolist(), vals))  # vqe.py:89
        if v == 0:
            term0 = np.array(vals)
        dims.append([len(x) for x in state.bond_vectors])
    set_shim(False)
    save("cfg2", {"mode": "O2 shim", "elapsed_s": time.perf_counter() - t0, "seed": w.meta["seed"]},
         energies=energies, terms_v0=term0, dims=np.array(dims, dtype=np.int64))


def gen_cfg3() -> None:
    from paper_1807_07914_b200.workloads import config3
    w = config3()
    rec = set_shim(True, record=True)
    t0 = time.perf_counter()
    state, bond_err = ref_evolve(w.programs[0], w.n, w.cutoff, w.max_bond, per_bond=True)
    t_ev = time.perf_counter() - t0
    keep, margin, gap = decision_margins(rec.spectra, w.cutoff, w.max_bond)
    t0 = time.perf_counter()
    z = np.array([state.expectation_pauli(p) for p in w.paulis])
    t_q = time.perf_counter() - t0
    z_env = to_oracle(state).expectations_env(w.paulis)
    norm = to_oracle(state).expectations_env(["I" * w.n])[0]
    set_shim(False)
    save("cfg3", {"mode": "O2 shim evolution + O2 expectation_pauli", "evolve_s": t_ev,
                  "query_s": t_q, "seed": w.meta["seed"]},
         z=z, z_env=z_env, norm=np.float64(norm), bond_err=bond_err, upd_keep=keep,
         upd_margin=margin, upd_gap=gap, **state_summary(state))


def _cfg4_circuit(c: int):
    """One cfg4 circuit through the O2-shimmed reference (a Pool task)."""
    from threadpoolctl import threadpool_limits
    from paper_1807_07914_b200.workloads import config4
    threadpool_limits(1)
    w = config4(circuits=c + 1, indices=[c])
    rec = set_shim(True, record=True)
    note = ""
    try:
        state, _ = ref_evolve(w.programs[0], w.n, w.cutoff, w.max_bond)
    except RuntimeError as exc:
        # LAPACK zgesdd occasionally reports non-convergence ("SVD failed on bond q",
        # mps.py:115-118) for one particular rounding of theta; the verbatim reference
        # (its own einsums, O1) evolves the same circuit fine, so pin that run instead
        note = f"O2 shim at 1 thread: {exc}; evolved verbatim (O1)"
        rec = set_shim(False, record=True)
        state, _ = ref_evolve(w.programs[0], w.n, w.cutoff, w.max_bond)
        set_shim(True)
    _, margin, gap = decision_margins(rec.spectra, w.cutoff, w.max_bond)
    out = (state.expectation_pauli(w.paulis[0]), [state.amplitude(b) for b in w.bitstrings[0]],
           [len(x) for x in state.bond_vectors], state.trunc_error_sq, state.max_bond_seen,
           state.peak_entries, float(margin.min()), float(gap.min()), note)
    set_shim(False)
    return out


def gen_cfg4(count: int = 1024) -> None:
    """All ``count`` circuits of cfg4 (circuit i depends on (seed, i) only, so these pin
    every prefix slice the bench and the tests run), one circuit per Pool task with
    single-threaded OpenBLAS."""
    import multiprocessing as mp
    from paper_1807_07914_b200.workloads import config4
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(os.cpu_count()) as pool:
        res = pool.map(_cfg4_circuit, range(count), chunksize=4)
    zz, amps, dims, errs, mbs, peaks, margins, gaps, fails = (list(x) for x in zip(*res))
    failed = [i for i, f in enumerate(fails) if f]
    save("cfg4", {"mode": "O2 shim", "circuits": count, "elapsed_s": time.perf_counter() - t0,
                  "seed": config4(circuits=1).meta["seed"],
                  "reference_retries": {str(i): fails[i] for i in failed}},
         zz=np.array(zz), amps=np.array(amps), dims=np.array(dims, dtype=np.int16),
         trunc_error_sq=np.array(errs), max_bond_seen=np.array(mbs, dtype=np.int64),
         peak_entries=np.array(peaks, dtype=np.int64), min_margin=np.array(margins),
         min_gap=np.array(gaps))


def gen_o2check() -> None:
    """Validate the O2 shim against the verbatim reference on one cfg4 circuit."""
    from paper_1807_07914_b200.workloads import config4
    w = config4(circuits=1)
    res = {}
    for mode in ("O1", "O2"):
        set_shim(mode == "O2")
        t0 = time.perf_counter()
        state, _ = ref_evolve(w.programs[0], w.n, w.cutoff, w.max_bond)
        zz = state.expectation_pauli(w.paulis[0])
        amps = np.array([state.amplitude(b) for b in w.bitstrings[0]])
        res[mode] = (zz, amps, [len(x) for x in state.bond_vectors], time.perf_counter() - t0)
    set_shim(False)
    rel_zz = abs(res["O1"][0] - res["O2"][0]) / abs(res["O1"][0])
    amp_err = np.max(np.abs(res["O1"][1] - res["O2"][1])) / np.max(np.abs(res["O1"][1]))
    meta = {"rel_zz": rel_zz, "amp_err_of_max": float(amp_err),
            "dims_equal": res["O1"][2] == res["O2"][2], "O1_s": res["O1"][3], "O2_s": res["O2"][3]}
    print(json.dumps(meta))
    (GOLDEN / "o2check.json").write_text(json.dumps(meta, indent=1))


def gen_cfg5() -> None:
    from paper_1807_07914_b200.workloads import config5
    w = config5()
    rec = set_shim(True, record=True)
    t0 = time.perf_counter()
    state, bond_err = ref_evolve(w.programs[0], w.n, w.cutoff, w.max_bond, per_bond=True)
    t_ev = time.perf_counter() - t0
    keep, margin, gap = decision_margins(rec.spectra, w.cutoff, w.max_bond)
    set_shim(False)
    t0 = time.perf_counter()
    vals = to_oracle(state).expectations_env(w.paulis + ["I" * w.n])
    t_q = time.perf_counter() - t0
    summ = state_summary(state)
    dims = summ["dims"]
    lam_head = np.stack([np.pad(v[:8], (0, 8 - min(8, len(v)))) for v in state.bond_vectors])
    save("cfg5", {"mode": "O2 shim evolution + O2+ env-reuse queries", "evolve_s": t_ev,
                  "query_s": t_q, "seed": w.meta["seed"]},
         x=vals[: w.n], z=vals[w.n: 2 * w.n], norm=np.float64(vals[-1]), bond_err=bond_err,
         dims=dims, lam_head=lam_head, lam=summ["lam"], trunc_error_sq=summ["trunc_error_sq"],
         max_bond_seen=summ["max_bond_seen"], peak_entries=summ["peak_entries"],
         upd_keep=keep, upd_margin=margin, upd_gap=gap)


if __name__ == "__main__":
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    table = {"small": gen_small, "cfg1": gen_cfg1, "cfg2": gen_cfg2, "cfg3": gen_cfg3,
             "cfg4": gen_cfg4, "cfg5": gen_cfg5, "o2check": gen_o2check}
    for arg in sys.argv[1:] or ["small"]:
        t0 = time.perf_counter()
        table[arg]()
        print(f"{arg}: {time.perf_counter() - t0:.1f} s", flush=True)
