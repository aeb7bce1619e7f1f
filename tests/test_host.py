"""Host-side logic on CPU: IR/gates/policy mirror the reference, lowering and
layer scheduling, the C ABI library loads and exports every header symbol, and
the product path refuses to run without a GPU (no CPU fallback)."""

import re
from pathlib import Path

import numpy as np
import pytest

from paper_1807_07914_b200 import (
    GateKind, Instruction, IrError, MatrixGate, SWAP_MATRIX, TruncationPolicy, check_unitary,
    compile_batch, gate_matrix, num_qubits,
)
from paper_1807_07914_b200 import _native
from paper_1807_07914_b200.engine import asap_layers, lower_program
from paper_1807_07914_b200.workloads import brick_circuit, config4, haar_unitary, random_program

ROOT = Path(__file__).resolve().parent.parent


def test_gate_conventions_match_oracle():
    from oracle.mps_oracle import oracle_gate_matrix
    rng = np.random.default_rng(3)
    for op in random_program(5, 200, rng):
        np.testing.assert_array_equal(gate_matrix(op), oracle_gate_matrix(op))
    cnot = gate_matrix(Instruction(GateKind.CNOT, (0, 1)))
    assert cnot[3, 2] == 1 and cnot[2, 3] == 1 and cnot[0, 0] == 1


def test_check_unitary():
    check_unitary(SWAP_MATRIX)
    with pytest.raises(ValueError, match="unitary"):
        check_unitary(np.diag([1.0, 2.0]))
    with pytest.raises(ValueError):
        check_unitary(np.eye(3))


def test_ir_validation():
    with pytest.raises(IrError):
        Instruction(GateKind.CNOT, (0,))
    with pytest.raises(IrError):
        Instruction(GateKind.CNOT, (1, 1))
    with pytest.raises(IrError):
        Instruction(GateKind.RX, (0,))
    with pytest.raises(IrError):
        MatrixGate(np.eye(2), (0, 1))
    assert num_qubits([Instruction(GateKind.X, (4,))]) == 5


def test_policy_validation_and_keep():
    with pytest.raises(ValueError):
        TruncationPolicy(cutoff=-1)
    with pytest.raises(ValueError):
        TruncationPolicy(max_bond=0)
    s = np.array([1.0, 0.5, 0.3, 1e-9])
    assert TruncationPolicy(1e-4, 2).keep_count(s) == 2
    assert TruncationPolicy(1e-4).keep_count(s) == 3
    c = TruncationPolicy(1e-10, 256, False).as_c()
    assert (c.cutoff, c.max_bond, c.relative) == (1e-10, 256, 0)


def test_lowering_routes_like_reference():
    # CNOT(4, 1): higher index moved down by SWAPs at 3, 2; gate SWAP.G.SWAP at 1; SWAPs back
    prog = [Instruction(GateKind.CNOT, (4, 1))]
    ar, site, mats = lower_program(prog, 6)
    assert ar.tolist() == [2, 2, 2, 2, 2]
    assert site.tolist() == [3, 2, 1, 2, 3]
    g = gate_matrix(prog[0])
    np.testing.assert_array_equal(mats[2], SWAP_MATRIX @ g @ SWAP_MATRIX)
    with pytest.raises(ValueError):
        lower_program([Instruction(GateKind.X, (6,))], 6)


def test_asap_layers_are_site_disjoint_and_ordered():
    rng = np.random.default_rng(9)
    prog = random_program(9, 300, rng)
    ar, site, _ = lower_program(prog, 9)
    lay = asap_layers(ar, site, 9)
    for L in range(lay.max() + 1):
        used = []
        for i in np.nonzero(lay == L)[0]:
            used += [site[i]] if ar[i] == 1 else [site[i], site[i] + 1]
        assert len(used) == len(set(used))
    last = {}
    for i in range(len(ar)):
        for q in ([site[i]] if ar[i] == 1 else [site[i], site[i] + 1]):
            assert lay[i] > last.get(q, -1)
            last[q] = lay[i]


def test_compile_batch_records_in_program_order():
    w = config4(circuits=3)
    plan = compile_batch(w.programs, w.n)
    assert plan.n_records == sum(sum(1 for op in p if len(op.qubits) == 2) for p in w.programs)
    assert plan.ranges.tolist() == [[0, 0, 372], [1, 372, 372], [2, 744, 372]]
    assert sorted(plan.logidx2.tolist()) == list(range(plan.n_records))
    # within a state, layer order never reverses program order of records on a site
    for s in range(3):
        sel = plan.items2[:, 0] == s
        assert np.all(np.diff(plan.logidx2[sel][np.argsort(plan.logidx2[sel])]) == 1)


def test_workload_generators_deterministic():
    a = brick_circuit(6, 3, np.random.default_rng(1))
    b = brick_circuit(6, 3, np.random.default_rng(1))
    assert [(o.kind, o.qubits, o.params) for o in a] == [(o.kind, o.qubits, o.params) for o in b]
    u = haar_unitary(np.random.default_rng(2))
    check_unitary(u)


def _header_functions():
    text = (ROOT / "include" / "bmps.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int32_t|int64_t|size_t|uint64_t|void|const char\*)\s+(bmps_\w+)\(", text, re.M)))


def test_library_exports_every_header_symbol():
    from paper_1807_07914_b200 import build
    build.build()
    lib = _native.load()
    declared = _header_functions()
    assert len(declared) >= 10
    for name in declared:
        assert hasattr(lib, name), name
        assert name in _native.EXPORTED, f"{name} missing from the ctypes signature table"
    assert lib.bmps_version() == 2
    assert lib.bmps_status_string(1).decode().startswith("SVD failed")
    assert lib.bmps_apply_2q_workspace_bytes(256, 4) > 4 * 2 * 4 * 256 * 256 * 16
    # per-call tunables: defaults come from the library, unknown names are rejected
    d = _native.default_params()
    assert d["tol_factor"] == 4.0 and d["jacobi_mode"] == 4 and d["block_w2"] == 32
    assert (d["thr_a"], d["thr_a_sweeps"], d["thr_b"], d["thr_b_sweeps"]) == (3e-2, 2, 3e-3, 5)
    with pytest.raises(ValueError):
        _native.params(nonsense=1)
    with _native.tunables(jac_cluster=4):
        assert _native.params().jac_cluster == 4
    assert _native.params().jac_cluster == -1


def test_library_exports_only_the_c_abi():
    """libbmps.so's dynamic symbol table holds the bmps_* entry points only (the
    statically linked CUDA runtime stays internal: version script csrc/libbmps.map)."""
    import subprocess
    from paper_1807_07914_b200 import build
    so = build.build()
    out = subprocess.run(["nm", "-D", "--defined-only", str(so)], capture_output=True, text=True,
                         check=True).stdout
    names = [ln.split()[-1] for ln in out.splitlines() if ln.strip()]
    assert names and all(n.startswith("bmps_") for n in names), [n for n in names if not n.startswith("bmps_")][:10]
    assert set(_header_functions()) <= set(names)


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1807_07914_b200 import MpsState
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        MpsState(3)


def test_product_path_never_imports_oracle():
    pkg = ROOT / "paper_1807_07914_b200"
    for f in pkg.rglob("*.py"):
        text = f.read_text()
        assert "from oracle" not in text and "import oracle" not in text, f


def test_reference_instruction_objects_are_accepted():
    """Duck typing: programs built with the reference's own mpsqvm.ir lower identically."""
    import sys
    ref_src = "/root/reference/pkg/src"
    if not Path(ref_src).exists():
        pytest.skip("reference not mounted (GPU box)")
    sys.path.insert(0, ref_src)
    sys.dont_write_bytecode = True
    try:
        import mpsqvm
        rng = np.random.default_rng(4)
        ours = random_program(6, 50, rng)
        theirs = [mpsqvm.Instruction(mpsqvm.GateKind(o.kind.value), o.qubits, o.params) for o in ours]
        a1, s1, m1 = lower_program(ours, 6)
        a2, s2, m2 = lower_program(theirs, 6)
        assert a1.tolist() == a2.tolist() and s1.tolist() == s2.tolist()
        for x, y in zip(m1, m2):
            np.testing.assert_array_equal(x, y)
        from mpsqvm.gates import gate_matrix as ref_gate_matrix
        for o in theirs:
            np.testing.assert_array_equal(gate_matrix(o), ref_gate_matrix(o))
    finally:
        sys.path.remove(ref_src)


def _python_plan(programs, n):
    """compile_batch restated with the Python lowering/layering (the readable spec)."""
    lay_l, st_l, ar_l, site_l, mat_l, rec_l, ranges, rb = [], [], [], [], [], [], [], 0
    for s, prog in enumerate(programs):
        ar, st, mats = lower_program(prog, n)
        lay = asap_layers(ar, st, n)
        two = ar == 2
        rec = np.full(len(ar), -1, dtype=np.int64)
        n2 = int(two.sum())
        rec[two] = rb + np.arange(n2)
        if n2:
            ranges.append((s, rb, n2))
        rb += n2
        lay_l.append(lay); st_l.append(np.full(len(ar), s, np.int32)); ar_l.append(ar)
        site_l.append(st); mat_l.extend(mats); rec_l.append(rec)
    layer, state, ar = np.concatenate(lay_l), np.concatenate(st_l), np.concatenate(ar_l)
    site, rec = np.concatenate(site_l), np.concatenate(rec_l)
    order = np.argsort(layer, kind="stable")
    one, two = order[ar[order] == 1], order[ar[order] == 2]
    return dict(n_layers=int(layer.max()) + 1,
                items1=np.stack([state[one], site[one]], 1), items2=np.stack([state[two], site[two]], 1),
                gates1=np.array([mat_l[i] for i in one]).reshape(-1, 2, 2),
                gates2=np.array([mat_l[i] for i in two]).reshape(-1, 4, 4),
                logidx2=rec[two], ranges=np.array(ranges).reshape(-1, 3))


def test_native_planner_matches_python_lowering_bit_for_bit():
    rng = np.random.default_rng(11)
    progs = [random_program(9, 150, rng) for _ in range(12)] + [[]]
    progs += [[MatrixGate(haar_unitary(rng), (5, 2)), Instruction(GateKind.RZ, (3,), (0.25,)),
               MatrixGate(haar_unitary(rng, 2), (1,)), Instruction(GateKind.MEASURE, (0,), (), 0)]]
    progs += [brick_circuit(9, 6, rng, haar_prob=0.5)]
    ref = _python_plan(progs, 9)
    plan = compile_batch(progs, 9)
    assert plan.n_layers == ref["n_layers"]
    for key in ("items1", "items2", "logidx2", "ranges"):
        np.testing.assert_array_equal(getattr(plan, key), ref[key], err_msg=key)
    for key in ("gates1", "gates2"):   # identical bits, not just close
        np.testing.assert_array_equal(getattr(plan, key).view(np.uint64), ref[key].view(np.uint64),
                                      err_msg=key)


def test_native_planner_errors_match_reference_messages():
    with pytest.raises(ValueError, match="site 7 out of range for 6 qubits"):
        compile_batch([[Instruction(GateKind.X, (1,))], [Instruction(GateKind.CNOT, (2, 7))]], 6)
    with pytest.raises(ValueError, match="distinct"):
        compile_batch([[Instruction(GateKind.CZ, (3, 3))]], 6)
    with pytest.raises(ValueError, match="not unitary"):
        compile_batch([[MatrixGate(np.ones((2, 2)), (0,))]], 2)


def test_compile_batch_rejects_duplicate_or_negative_states():
    """one program per state per plan (the layering and the in-order stats
    replay assume it); duplicates or negative indices are a ValueError, and a plan
    that addresses a state beyond the batch is refused by MpsBatch.execute."""
    progs = [brick_circuit(4, 2, np.random.default_rng(k)) for k in range(3)]
    with pytest.raises(ValueError, match="distinct"):
        compile_batch(progs, 4, states=[0, 1, 0])
    with pytest.raises(ValueError, match="distinct"):
        compile_batch(progs, 4, states=[0, -1, 2])
    with pytest.raises(ValueError, match="state indices"):
        compile_batch(progs, 4, states=[0, 1])
    assert compile_batch(progs, 4, states=[5, 1, 3]).max_state == 5


def test_simulate_batch_slice_schedule_covers_every_circuit_once():
    """simulate_batch's default slices (small first slice, doubling, quarters) and the
    fixed-size ones tile [0, S) exactly."""
    from paper_1807_07914_b200.backends import slice_schedule
    for S in (0, 1, 255, 256, 300, 512, 1000, 1024, 4096):
        for chunk in (None, 1, 100, 5000):
            sl = slice_schedule(S, chunk)
            assert sum(b - a for a, b in sl) == S
            assert all(a < b for a, b in sl)
            assert all(sl[i][1] == sl[i + 1][0] for i in range(len(sl) - 1))
            assert not sl or (sl[0][0] == 0 and sl[-1][1] == S)
    assert slice_schedule(1024) == [(0, 64), (64, 192), (192, 448), (448, 704), (704, 1024)]
    assert slice_schedule(200) == [(0, 200)]


def test_uniform_batch_extraction_equals_per_op_extraction():
    """The planner's fast path for batches of one circuit structure (a bound VQE ansatz,
    config 2) yields exactly the arrays of the per-op loop; mixed batches, MEASUREs and
    matrix gates are handled (or declined) the same way."""
    import numpy as np
    from paper_1807_07914_b200 import engine, workloads as W
    from paper_1807_07914_b200.ir import GateKind, Instruction, MatrixGate

    def same(a, b):
        for x, y in zip(a, b):
            if isinstance(x, np.ndarray):
                assert x.dtype == y.dtype and np.array_equal(x, y)
            else:
                assert x == y

    progs = W.config2(batch=6).programs
    fast = engine._extract_uniform(progs)
    assert fast is not None
    same(fast, engine._extract_slow(progs))
    with_measure = [list(p) + [Instruction(GateKind.MEASURE, (0,))] for p in progs]
    fast = engine._extract_uniform(with_measure)
    assert fast is not None
    same(fast, engine._extract_slow(with_measure))
    mixed = list(progs[:5]) + [list(progs[5])[:-1]]
    assert engine._extract_uniform(mixed) is None
    swapped = list(progs[:5]) + [list(progs[5])[:-1] + [Instruction(GateKind.CZ, (0, 1))]]
    assert engine._extract_uniform(swapped) is None
    same(engine._extract(swapped), engine._extract_slow(swapped))
    custom = [list(p) + [MatrixGate(np.eye(2, dtype=complex), (0,))] for p in progs]
    assert engine._extract_uniform(custom) is None
    # whole plans agree too
    p_fast = engine.compile_batch(progs, 20)
    engine._UNIFORM_FAST = False
    try:
        p_slow = engine.compile_batch(progs, 20)
    finally:
        engine._UNIFORM_FAST = True
    for name in ("items1", "items2", "off1", "off2", "logidx2", "ranges", "gates1", "gates2"):
        assert np.array_equal(getattr(p_fast, name), getattr(p_slow, name))
