"""Rebuild the reference-parsed kernel trees of tests/golden/frontend.json
(oracle/gen_frontend.py) with this package's IR classes."""

import json

from conftest import GOLDEN

from paper_1807_07914_b200 import CompositeInstruction, GateKind, Instruction, PauliHamiltonian


def load_frontend():
    return json.loads((GOLDEN / "frontend.json").read_text())


def tree_from_json(d):
    if "kind" in d:
        return Instruction(GateKind(d["kind"]), tuple(d["qubits"]), tuple(d["params"]),
                           d["classical_target"])
    return CompositeInstruction(d["name"], tuple(d["formal_params"]),
                                tuple(tree_from_json(c) for c in d["children"]),
                                None if d["call_args"] is None else tuple(d["call_args"]))


def hamiltonian(fx):
    return PauliHamiltonian(tuple(zip(fx["coeffs"], fx["paulis"])))
