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


def set_shim(on: bool) -> None:
    _, ref_mps = _ref()
    if on:
        shim = _NpShim("numpy_o2")
        shim.einsum = lambda *a, **k: np.einsum(*a, **{**k, "optimize": True})
        ref_mps.np = shim
    else:
        ref_mps.np = np


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
    set_shim(False)
    t0 = time.perf_counter()
    state, _ = ref_evolve(w.programs[0], w.n, w.cutoff, w.max_bond)
    t_ev = time.perf_counter() - t0
    amps = np.array([state.amplitude(b) for b in w.bitstrings[0]])
    set_shim(True)
    t0 = time.perf_counter()
    z = np.array([state.expectation_pauli(p) for p in w.paulis])
    t_q = time.perf_counter() - t0
    set_shim(False)
    save("cfg1", {"mode": "O1 evolution + amplitudes; O2 shim for <Z>", "evolve_s": t_ev,
                  "query_s": t_q, "seed": w.meta["seed"]},
         amps=amps, z=z, **state_summary(state))


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
    set_shim(True)
    t0 = time.perf_counter()
    state, bond_err = ref_evolve(w.programs[0], w.n, w.cutoff, w.max_bond, per_bond=True)
    t_ev = time.perf_counter() - t0
    t0 = time.perf_counter()
    z = np.array([state.expectation_pauli(p) for p in w.paulis])
    t_q = time.perf_counter() - t0
    z_env = to_oracle(state).expectations_env(w.paulis)
    norm = to_oracle(state).expectations_env(["I" * w.n])[0]
    set_shim(False)
    save("cfg3", {"mode": "O2 shim evolution + O2 expectation_pauli", "evolve_s": t_ev,
                  "query_s": t_q, "seed": w.meta["seed"]},
         z=z, z_env=z_env, norm=np.float64(norm), bond_err=bond_err, **state_summary(state))


def gen_cfg4(count: int = 16) -> None:
    from paper_1807_07914_b200.workloads import config4
    w = config4()
    set_shim(True)
    zz, amps, dims, errs, mbs = [], [], [], [], []
    t0 = time.perf_counter()
    for c in range(count):
        state, _ = ref_evolve(w.programs[c], w.n, w.cutoff, w.max_bond)
        zz.append(state.expectation_pauli(w.paulis[0]))
        amps.append([state.amplitude(b) for b in w.bitstrings[c]])
        dims.append([len(x) for x in state.bond_vectors])
        errs.append(state.trunc_error_sq)
        mbs.append(state.max_bond_seen)
    set_shim(False)
    save("cfg4", {"mode": "O2 shim", "circuits": count, "elapsed_s": time.perf_counter() - t0,
                  "seed": w.meta["seed"]},
         zz=np.array(zz), amps=np.array(amps), dims=np.array(dims, dtype=np.int64),
         trunc_error_sq=np.array(errs), max_bond_seen=np.array(mbs, dtype=np.int64))


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
    set_shim(True)
    t0 = time.perf_counter()
    state, bond_err = ref_evolve(w.programs[0], w.n, w.cutoff, w.max_bond, per_bond=True)
    t_ev = time.perf_counter() - t0
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
         dims=dims, lam_head=lam_head, trunc_error_sq=summ["trunc_error_sq"],
         max_bond_seen=summ["max_bond_seen"], peak_entries=summ["peak_entries"])


if __name__ == "__main__":
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    table = {"small": gen_small, "cfg1": gen_cfg1, "cfg2": gen_cfg2, "cfg3": gen_cfg3,
             "cfg4": gen_cfg4, "cfg5": gen_cfg5, "o2check": gen_o2check}
    for arg in sys.argv[1:] or ["small"]:
        t0 = time.perf_counter()
        table[arg]()
        print(f"{arg}: {time.perf_counter() - t0:.1f} s", flush=True)
