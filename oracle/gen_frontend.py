"""Front-end fixtures from the REFERENCE itself -- TEST INFRASTRUCTURE ONLY.

SURVEY §8(f) row 3: kernel-language text -> ``parse`` (``R:src/mpsqvm/parser.py:242``)
-> ``bind_parameters`` -> ``flatten`` (``R:src/mpsqvm/ir.py:150-184``) -> the MPS
executor, plus the multi-parameter sweep. The reference parser cannot travel to
the GPU box, so this script (run in the build container, where
``/root/reference`` is mounted read-only) parses the kernels below with the
reference, serialises the parsed kernel TREES (composite nodes, call sites,
symbolic parameter slots) to ``tests/golden/frontend.json``, and records the
reference's own answers:

* ``vqe.sweep`` of the one-parameter kernel (the reference driver, ``vqe.py:100-125``);
* for each parameter vector of the multi-parameter kernel: the reference's
  ``bind_parameters`` + ``flatten`` + ``run_program(backend="mps")`` and the
  energy ``sum_k c_k <P_k>`` (``vqe.py:87-89``), plus amplitudes.

On the GPU box ``tests/test_gpu_frontend.py`` rebuilds the trees with this
package's IR classes, binds and flattens them with this package's
``bind_parameters`` / ``flatten`` and runs them through the GPU executor.

Usage: ``python -m oracle.gen_frontend``.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF_SRC = "/root/reference/pkg/src"
ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "tests" / "golden" / "frontend.json"
sys.dont_write_bytecode = True

# Kernel text written for this fixture in the reference's kernel language:
# nested calls with literal and symbolic arguments, non-adjacent two-qubit gates
# (SWAP routing), MEASUREs (dropped by the driver), every gate kind.
KERNELS = """
# one entangling layer, two angles
__qpu__ layer(AcceleratorBuffer b, double a, double c) {
  RY(a) 0
  RY(c) 1
  RY(a) 2
  RY(c) 3
  CNOT 0 1
  CNOT 2 3
  CZ 1 2
}
__qpu__ ansatz(AcceleratorBuffer b, double t0, double t1, double t2, double t3) {
  H 0
  H 3
  layer(b, t0, t1)
  RZ(t2) 2
  CNOT 0 3
  layer(b, t3, 0.125)
  SWAP 1 4
  RX(t1) 4
  CNOT 4 1
  X 5
  Y 2
  Z 1
  I 0
  RZ(t3) 5
  CNOT 5 2
  MEASURE 0 [0]
}
__qpu__ single(AcceleratorBuffer b, double t0) {
  H 0
  CNOT 0 1
  RY(t0) 1
  CNOT 1 2
  RX(t0) 2
  CNOT 0 2
  MEASURE 1 [0]
}
"""
N = 6


def _ref():
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import mpsqvm
    return mpsqvm


def tree_to_json(node):
    """Parsed reference tree -> JSON (leaves: kind, qubits, params, classical_target)."""
    if hasattr(node, "kind"):
        return {"kind": node.kind.value, "qubits": list(node.qubits), "params": list(node.params),
                "classical_target": node.classical_target}
    return {"name": node.name, "formal_params": list(node.formal_params),
            "call_args": None if node.call_args is None else list(node.call_args),
            "children": [tree_to_json(c) for c in node.children]}


def main() -> None:
    mp = _ref()
    from mpsqvm import vqe as rvqe
    from mpsqvm.backends import run_program
    from mpsqvm.hamiltonian import PauliHamiltonian
    from mpsqvm.ir import bind_parameters, flatten
    from mpsqvm.mps import TruncationPolicy
    from mpsqvm.parser import parse

    unit = parse(KERNELS)
    rng = np.random.default_rng(1807)
    paulis, coeffs = [], []
    for _ in range(14):
        w = int(rng.integers(1, 4))
        sup = rng.choice(N, size=w, replace=False)
        ch = ["I"] * N
        for q in sup:
            ch[int(q)] = "XYZ"[int(rng.integers(3))]
        paulis.append("".join(ch))
        coeffs.append(float(rng.standard_normal()))
    paulis.append("I" * N)
    coeffs.append(0.75)
    ham = PauliHamiltonian(tuple(zip(coeffs, paulis)))
    policies = [(0.0, None), (1e-3, 2)]
    vectors = rng.uniform(-np.pi, np.pi, size=(6, 4))
    bits = ["".join("01"[int(b)] for b in rng.integers(0, 2, N)) for _ in range(8)]
    multi = []
    for cutoff, max_bond in policies:
        pol = TruncationPolicy(cutoff, max_bond)
        energies, amps, dims = [], [], []
        for vec in vectors:
            prog = [i for i in flatten(bind_parameters(unit.kernels["ansatz"], list(vec)))
                    if i.kind is not mp.GateKind.MEASURE]
            st = run_program(prog, N, "mps", pol)
            energies.append(sum(c * st.expectation_pauli(p) for c, p in ham.terms))   # vqe.py:89
            amps.append([[st.amplitude(b).real, st.amplitude(b).imag] for b in bits])
            dims.append([len(v) for v in st.bond_vectors])
        multi.append({"cutoff": cutoff, "max_bond": max_bond, "energies": energies,
                      "amps": amps, "dims": dims})
    sweeps = []
    for cutoff, max_bond in policies:
        res = rvqe.sweep(unit.kernels["single"], ham, -1.0, 2.0, 7, "mps",
                         TruncationPolicy(cutoff, max_bond))
        sweeps.append({"cutoff": cutoff, "max_bond": max_bond, "thetas": list(res.thetas),
                       "energies": list(res.energies), "argmin_theta": res.argmin_theta,
                       "min_energy": res.min_energy})
    out = {
        "generator": "oracle/gen_frontend.py (reference parse / bind_parameters / flatten / "
                     "run_program / vqe.sweep)",
        "text": KERNELS, "n": N,
        "kernels": {k: tree_to_json(v) for k, v in unit.kernels.items()},
        "paulis": paulis, "coeffs": coeffs, "vectors": vectors.tolist(), "bits": bits,
        "multi": multi, "sweeps": sweeps,
    }
    OUT.write_text(json.dumps(out, indent=1))
    print(f"wrote {OUT} ({OUT.stat().st_size} B)")


if __name__ == "__main__":
    main()
