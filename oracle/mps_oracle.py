"""Numpy restatement of the reference MPS algorithm -- TEST INFRASTRUCTURE ONLY.

Oracle for the B200 MPS hot path (see ``oracle/__init__.py`` for who may
import it). It restates ``R:src/mpsqvm/mps.py`` (``R:`` = ``/root/reference/pkg/``)
operation by operation, keeping every numerical decision of the reference:

* truncation rule ``TruncationPolicy.keep_count`` (``mps.py:43-49``);
* two-site update: theta absorbs lambda_{q-1}, lambda_q, lambda_{q+1}
  (``mps.py:101-109``), gate applied as ``g[a,b,s,t]`` (``:110-111``), matrix rows
  ``(l,a)`` / columns ``(b,r)`` (``:113-114``), thin SVD by LAPACK ``zgesdd``
  (``:116``), ``trunc_error_sq`` accumulated from the raw discarded values
  before renormalisation (``:120-127``), pseudo-inverse split with the strict
  ``> 1e-12`` floor (``:129-135``), stats after every update (``:82-84``);
* SWAP routing order (``mps.py:138-157``);
* queries on ``T_k = Gamma_k * lambda_k`` (``mps.py:165-170``): amplitude
  (``:172-179``), full left-to-right expectation sweep from ``[[1]]`` with no
  normalisation and the 1e-10 imaginary-residue check (``:188-204``).

Two contraction modes:

* ``verbatim=True`` issues the reference's own ``np.einsum`` calls (numpy's
  default ``optimize=False``), so timing it measures the reference CPU path;
* ``verbatim=False`` (default) evaluates the same sums with BLAS matmuls and
  ``einsum(optimize=True)`` (the SURVEY §8(c) "O2" shim) -- identical algorithm,
  different summation order, orders of magnitude faster at chi >= 64.

``expectations_env`` evaluates many Pauli strings with cached left/right
identity environments: the ``mps.py:196-204`` sum reassociated (SURVEY §8(c)
"O2+"), no canonical-form assumption.

Parity pin: ``tests/test_oracle.py`` checks this module against golden
vectors produced by the reference itself (``oracle/gen_golden.py``).
"""

from __future__ import annotations

import numpy as np

PINV_FLOOR = 1e-12  # mps.py:21

_P = {
    "I": np.eye(2, dtype=complex),
    "X": np.array([[0, 1], [1, 0]], dtype=complex),
    "Y": np.array([[0, -1j], [1j, 0]], dtype=complex),
    "Z": np.array([[1, 0], [0, -1]], dtype=complex),
}
_SWAP = np.eye(4, dtype=complex)[[0, 2, 1, 3]]
_SQ = 1.0 / np.sqrt(2.0)
_FIXED = {
    "I": _P["I"], "X": _P["X"], "Y": _P["Y"], "Z": _P["Z"],
    "H": np.array([[_SQ, _SQ], [_SQ, -_SQ]], dtype=complex),
    "CNOT": np.eye(4, dtype=complex)[[0, 1, 3, 2]],
    "CZ": np.diag([1, 1, 1, -1]).astype(complex),
    "SWAP": _SWAP,
}


def oracle_gate_matrix(op) -> np.ndarray:
    """Gate matrix per ``R:src/mpsqvm/gates.py:34-59`` (independent of the product code)."""
    m = getattr(op, "matrix", None)
    if m is not None:
        return np.asarray(m, dtype=complex)
    name = op.kind.value
    if name in _FIXED:
        return _FIXED[name]
    th = float(op.params[0])
    c, s = np.cos(th / 2), np.sin(th / 2)
    if name == "RX":
        return np.array([[c, -1j * s], [-1j * s, c]])
    if name == "RY":
        return np.array([[c, -s], [s, c]], dtype=complex)
    if name == "RZ":
        return np.diag([np.exp(-1j * th / 2), np.exp(1j * th / 2)])
    raise ValueError(f"{name} has no unitary matrix")


def keep_count(sigma: np.ndarray, cutoff: float, max_bond: int | None, relative: bool = True) -> int:
    """``TruncationPolicy.keep_count`` (mps.py:43-49)."""
    if cutoff > 0:
        thr = cutoff * (sigma[0] if relative else 1.0)
        k = int(np.count_nonzero(sigma >= thr))
    else:
        k = len(sigma)
    k = max(k, 1)
    return k if max_bond is None else min(k, max_bond)


def _pinv(lam: np.ndarray) -> np.ndarray:
    return np.where(lam > PINV_FLOOR, 1.0 / np.maximum(lam, PINV_FLOOR), 0.0)


class OracleMps:
    """Vidal-form MPS, |0...0> initially (``mps.py:55-66``)."""

    def __init__(self, n: int, cutoff: float = 1e-4, max_bond: int | None = None,
                 relative: bool = True, verbatim: bool = False):
        if n < 1:
            raise ValueError("need at least one qubit")
        self.n, self.cutoff, self.max_bond, self.relative = n, cutoff, max_bond, relative
        self.verbatim = verbatim
        self.gammas = [np.array([1.0, 0.0], dtype=complex).reshape(1, 2, 1) for _ in range(n)]
        self.lams = [np.ones(1) for _ in range(n - 1)]
        self.trunc_error_sq = 0.0
        self.max_bond_seen = 1
        self.peak_entries = 2 * n
        self.bond_trunc = np.zeros(max(n - 1, 0))  # per-bond discarded weight (cfg5 output)

    # -- bookkeeping (mps.py:70-84) ------------------------------------------
    def total_entries(self) -> int:
        return int(sum(g.size for g in self.gammas))

    def current_max_bond(self) -> int:
        return 1 if self.n == 1 else max(len(v) for v in self.lams)

    def dims(self) -> list[int]:
        return [len(v) for v in self.lams]

    # -- updates ---------------------------------------------------------------
    def apply_1q(self, g: np.ndarray, q: int) -> None:
        """mps.py:88-92."""
        t = self.gammas[q]
        if self.verbatim:
            self.gammas[q] = np.einsum("st,ltr->lsr", g, t)
        else:
            self.gammas[q] = np.einsum("st,ltr->lsr", g, t, optimize=True)

    def apply_2q(self, g: np.ndarray, q: int) -> None:
        """mps.py:94-136."""
        if q + 1 >= self.n:
            raise ValueError(f"site {q} has no right neighbour (n={self.n})")
        lam_l = self.lams[q - 1] if q > 0 else np.ones(1)
        lam_r = self.lams[q + 1] if q + 1 < self.n - 1 else np.ones(1)
        a, b, lam_m = self.gammas[q], self.gammas[q + 1], self.lams[q]
        dl, dm, dr = a.shape[0], a.shape[2], b.shape[2]
        if self.verbatim:
            th = np.einsum("l,lsm,m,mtr,r->lstr", lam_l, a, lam_m, b, lam_r)
            th = np.einsum("abst,lstr->labr", g.reshape(2, 2, 2, 2), th)
        else:
            left = (lam_l[:, None, None] * a * lam_m[None, None, :]).reshape(dl * 2, dm)
            right = (b * lam_r[None, None, :]).reshape(dm, 2 * dr)
            th = (left @ right).reshape(dl, 2, 2, dr)
            th = np.einsum("abst,lstr->labr", g.reshape(2, 2, 2, 2), th, optimize=True)
        mat = th.reshape(dl * 2, 2 * dr)
        try:
            u, s, vh = np.linalg.svd(mat, full_matrices=False)
        except np.linalg.LinAlgError as exc:  # mps.py:117-118
            raise RuntimeError(f"SVD failed on bond {q}") from exc
        k = keep_count(s, self.cutoff, self.max_bond, self.relative)
        dropped = float(np.sum(s[k:] ** 2))
        self.trunc_error_sq += dropped
        self.bond_trunc[q] += dropped
        s = s[:k]
        nrm = np.linalg.norm(s)
        if nrm == 0.0:
            raise RuntimeError(f"all singular values truncated on bond {q}")
        self.gammas[q] = _pinv(lam_l)[:, None, None] * u[:, :k].reshape(dl, 2, k)
        self.gammas[q + 1] = vh[:k, :].reshape(k, 2, dr) * _pinv(lam_r)[None, None, :]
        self.lams[q] = s / nrm
        self.peak_entries = max(self.peak_entries, self.total_entries())
        self.max_bond_seen = max(self.max_bond_seen, self.current_max_bond())

    def apply_routed(self, g: np.ndarray, q1: int, q2: int) -> None:
        """SWAP-chain routing, mps.py:138-157 (same order of adjacent updates)."""
        if q1 == q2:
            raise ValueError("two-qubit gate needs two distinct sites")
        lo, hi = min(q1, q2), max(q1, q2)
        for k in range(hi - 1, lo, -1):
            self.apply_2q(_SWAP, k)
        self.apply_2q(g if q1 < q2 else _SWAP @ g @ _SWAP, lo)
        for k in range(lo + 1, hi):
            self.apply_2q(_SWAP, k)

    def run(self, program) -> "OracleMps":
        """Per-gate loop of ``backends.mps_run`` (backends.py:47-60)."""
        for op in program:
            kind = getattr(op, "kind", None)
            if kind is not None and kind.value == "MEASURE":
                continue
            g = oracle_gate_matrix(op)
            if len(op.qubits) == 1:
                self.apply_1q(g, op.qubits[0])
            else:
                self.apply_routed(g, op.qubits[0], op.qubits[1])
        return self

    # -- queries ---------------------------------------------------------------
    def site_matrix(self, k: int) -> np.ndarray:
        """T_k = Gamma_k * lambda_k (mps.py:165-170)."""
        t = self.gammas[k]
        return t * self.lams[k][None, None, :] if k < self.n - 1 else t

    def amplitude(self, bits: str) -> complex:
        """mps.py:172-179."""
        if len(bits) != self.n or any(b not in "01" for b in bits):
            raise ValueError(f"need a bitstring of length {self.n}, got {bits!r}")
        vec = np.ones(1, dtype=complex)
        for k, b in enumerate(bits):
            vec = vec @ self.site_matrix(k)[:, int(b), :]
        return complex(vec[0])

    def _transfer(self, env: np.ndarray, k: int, label: str) -> np.ndarray:
        t = self.site_matrix(k)
        if self.verbatim:
            return np.einsum("ab,asr,st,btq->rq", env, t.conj(), _P[label], t)
        ot = np.einsum("st,btq->bsq", _P[label], t, optimize=True)
        f = np.tensordot(env, ot, axes=([1], [0]))          # f[a,s,q]
        return np.tensordot(t.conj(), f, axes=([0, 1], [0, 1]))  # e[r,q]

    def expectation(self, pauli: str) -> float:
        """Full left-to-right sweep, mps.py:188-204."""
        if len(pauli) != self.n:
            raise ValueError(f"Pauli string length {len(pauli)} != qubit count {self.n}")
        env = np.ones((1, 1), dtype=complex)
        for k, lab in enumerate(pauli):
            env = self._transfer(env, k, lab)
        val = complex(env[0, 0])
        if abs(val.imag) > 1e-10:
            raise RuntimeError(f"expectation has imaginary residue {val.imag:.3e}")
        return val.real

    def norm_sq(self) -> float:
        return self.expectation("I" * self.n)

    def _right_transfer(self, env: np.ndarray, k: int, label: str) -> np.ndarray:
        t = self.site_matrix(k)
        ot = np.einsum("st,btq->bsq", _P[label], t, optimize=True)
        f = np.tensordot(ot, env, axes=([2], [1]))           # f[b,s,r] = sum_q ot[b,s,q] env[r,q]
        return np.tensordot(t.conj(), f, axes=([1, 2], [1, 2]))  # e[a,b]

    def expectations_env(self, paulis: list[str]) -> np.ndarray:
        """Many strings with cached identity environments (mps.py:196-204 reassociated)."""
        n = self.n
        left = [np.ones((1, 1), dtype=complex)]
        for k in range(n):
            left.append(self._transfer(left[-1], k, "I"))
        right = [None] * (n + 1)
        right[n] = np.ones((1, 1), dtype=complex)
        for k in range(n - 1, -1, -1):
            right[k] = self._right_transfer(right[k + 1], k, "I")
        out = np.empty(len(paulis))
        for i, p in enumerate(paulis):
            sup = [k for k, c in enumerate(p) if c != "I"]
            if not sup:
                val = complex(np.sum(left[n]))
            else:
                env = left[sup[0]]
                for k in range(sup[0], sup[-1] + 1):
                    env = self._transfer(env, k, p[k])
                val = complex(np.sum(env * right[sup[-1] + 1]))
            if abs(val.imag) > 1e-10:
                raise RuntimeError(f"expectation has imaginary residue {val.imag:.3e}")
            out[i] = val.real
        return out


def oracle_sample(o: "OracleMps", shots: int, rng: np.random.Generator) -> dict[str, int]:
    """Sequential conditional sampling, mps.py:206-237 (one rng.random() per qubit per shot)."""
    counts: dict[str, int] = {}
    mats = [o.site_matrix(k) for k in range(o.n)]
    for _ in range(shots):
        vec = np.ones(1, dtype=complex)
        key = []
        for k in range(o.n):
            w0 = vec @ mats[k][:, 0, :]
            w1 = vec @ mats[k][:, 1, :]
            p0 = float(np.vdot(w0, w0).real)
            p1 = float(np.vdot(w1, w1).real)
            tot = p0 + p1
            pz = p0 / tot if tot > 0 else 0.5
            if rng.random() < pz:
                key.append("0")
                vec = w0
            else:
                key.append("1")
                vec = w1
        s = "".join(key)
        counts[s] = counts.get(s, 0) + 1
    return counts


def oracle_run(program, n: int, cutoff: float = 1e-4, max_bond: int | None = None,
               relative: bool = True, verbatim: bool = False) -> OracleMps:
    return OracleMps(n, cutoff, max_bond, relative, verbatim).run(program)
