"""Composite kernels -> bind_parameters -> flatten (R:src/mpsqvm/ir.py:86-184), the
front end that feeds the GPU layer compiler for parameter sweeps.
Host logic only: no GPU needed."""

import importlib.util
import math
import sys
from pathlib import Path

import pytest

from paper_1807_07914_b200 import (CompositeInstruction, GateKind, Instruction, IrError,
                                   bind_parameters, flatten)
from paper_1807_07914_b200.vqe import _basis_rotations, _unitary_program, binomial_sigma, sweep

I = Instruction


def nested_ansatz():
    inner = CompositeInstruction("layer", ("phi",), (
        I(GateKind.RZ, (1,), ("theta",)),
        I(GateKind.CNOT, (1, 2)),
        I(GateKind.RX, (2,), (0.25,)),
    ), call_args=("theta",))
    return CompositeInstruction("ansatz", ("theta",), (
        I(GateKind.H, (0,)),
        I(GateKind.RY, (0,), ("theta",)),
        inner,
        I(GateKind.MEASURE, (0,), (), 0),
        I(GateKind.RZ, (2,), ("theta",)),
    ))


def test_bind_then_flatten_preorder():
    a = nested_ansatz()
    b = bind_parameters(a, [0.5])
    assert b.formal_params == () and a.formal_params == ("theta",)   # input not mutated
    prog = flatten(b)
    assert [(i.kind.value, i.qubits) for i in prog] == [
        ("H", (0,)), ("RY", (0,)), ("RZ", (1,)), ("CNOT", (1, 2)), ("RX", (2,)),
        ("MEASURE", (0,)), ("RZ", (2,))]
    assert prog[1].params == (0.5,) and prog[2].params == (0.5,) and prog[6].params == (0.5,)
    assert b.children[2].call_args == (0.5,) and b.children[2].formal_params == ("phi",)
    # a callee's own formal is not bound by the caller's values (ir.py:133-147)
    own = CompositeInstruction("k", ("theta",), (CompositeInstruction(
        "c", ("phi",), (I(GateKind.RZ, (0,), ("phi",)),)),))
    with pytest.raises(IrError, match=r"unbound parameter\(s\) \['phi'\]"):
        flatten(bind_parameters(own, [1.0]))


def test_flatten_rejects_unbound_and_bind_checks_arity():
    a = nested_ansatz()
    with pytest.raises(IrError, match="unbound parameter"):
        flatten(a)
    with pytest.raises(IrError, match="takes 1 parameter"):
        bind_parameters(a, [1.0, 2.0])


def test_unitary_program_drops_measure_and_checks_formals():
    a = CompositeInstruction("k", ("t",), (I(GateKind.RX, (0,), ("t",)), I(GateKind.MEASURE, (0,))))
    prog = _unitary_program(a, 0.1)
    assert [i.kind for i in prog] == [GateKind.RX] and prog[0].params == (0.1,)
    two = CompositeInstruction("k2", ("a", "b"), ())
    with pytest.raises(ValueError, match="exactly one formal parameter"):
        _unitary_program(two, 0.0)
    with pytest.raises(ValueError, match="at least 2 points"):
        sweep(a, None, count=1)


def test_basis_rotations_and_sigma():
    rot = _basis_rotations("XIYZ")
    assert [(i.kind, i.qubits, i.params) for i in rot] == [
        (GateKind.H, (0,), ()), (GateKind.RZ, (2,), (-math.pi / 2,)), (GateKind.H, (2,), ())]
    assert binomial_sigma(1.0, 100) == 0.0 and abs(binomial_sigma(0.0, 100) - 0.1) < 1e-15


REF = Path("/root/reference/pkg/src")


@pytest.mark.skipif(not REF.exists(), reason="reference tree not present")
def test_matches_reference_bind_flatten_on_reference_objects():
    """Trees built from the reference's own classes flatten to the same gates."""
    sys.path.insert(0, str(REF))
    try:
        rir = importlib.import_module("mpsqvm.ir")
    finally:
        sys.path.remove(str(REF))
    K = rir.GateKind
    inner = rir.CompositeInstruction("layer", ("phi",), (
        rir.Instruction(K.RZ, (1,), ("theta",)), rir.Instruction(K.CZ, (1, 2))), ("theta",))
    root = rir.CompositeInstruction("ansatz", ("theta",), (
        rir.Instruction(K.RY, (0,), ("theta",)), inner, rir.Instruction(K.SWAP, (0, 2))))
    ref = rir.flatten(rir.bind_parameters(root, [0.75]))
    ours = flatten(bind_parameters(root, [0.75]))
    assert [(i.kind.value, i.qubits, i.params) for i in ref] == \
        [(i.kind.value, i.qubits, i.params) for i in ours]


def test_frontend_fixture_is_the_reference_parse():
    """tests/golden/frontend.json holds exactly what the reference parser produces for
    its kernel text, and this package's bind/flatten of the rebuilt trees equal the
    reference's (runs where /root/reference is mounted; the GPU box uses the fixture)."""
    import json
    ref_src = "/root/reference/pkg/src"
    if not Path(ref_src).exists():
        pytest.skip("reference not mounted (GPU box)")
    sys.path.insert(0, ref_src)
    sys.dont_write_bytecode = True
    from mpsqvm.ir import bind_parameters as rbind, flatten as rflatten
    from mpsqvm.parser import parse
    from frontend_fixture import load_frontend, tree_from_json
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "oracle"))
    from gen_frontend import tree_to_json
    fx = load_frontend()
    unit = parse(fx["text"])
    assert {k: tree_to_json(v) for k, v in unit.kernels.items()} == fx["kernels"]
    for vec in fx["vectors"]:
        theirs = rflatten(rbind(unit.kernels["ansatz"], list(vec)))
        ours = flatten(bind_parameters(tree_from_json(fx["kernels"]["ansatz"]), list(vec)))
        assert [(i.kind.value, tuple(i.qubits), tuple(i.params)) for i in ours] == \
               [(i.kind.value, tuple(i.qubits), tuple(i.params)) for i in theirs]
