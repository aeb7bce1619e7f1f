"""Device-resident MPS state batches and the layered program executor.

``MpsBatch`` owns S independent n-qubit Vidal-form states in HBM (torch
tensors used only as device buffers) and drives ``libbmps.so`` through its C
ABI. Programs are lowered exactly like the reference's per-gate loop
(``R:src/mpsqvm/backends.py:47-60``, SWAP routing ``R:src/mpsqvm/mps.py:138-157``)
and then scheduled ASAP into layers of site-disjoint operations: in Vidal form
a two-site update on (q, q+1) reads bonds q-1..q+1 and writes Gamma_q,
Gamma_{q+1}, lambda_q only, so ops sharing no site commute bit-exactly and one
layer (over all S states) is one batched launch sequence. Bookkeeping
(``trunc_error_sq``, ``peak_entries``, ``max_bond_seen``; ``mps.py:82-84``) is
replayed on the device in program order, so it matches the sequential
reference regardless of the schedule.

Host code never reads device state while a program runs: bond dimensions stay
on the device, and the host only keeps an upper-bound model
(``dim_ub[s, b] <= min(2 dim_ub[s, b-1], 2 dim_ub[s, b+1], max_bond)``) to size
grids and grow the capacity.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from math import cos, sin

import numpy as np
import torch

from . import _native
from .gates import SWAP_MATRIX, check_unitary, gate_matrix
from .hamiltonian import encode_paulis
from .policy import TruncationPolicy

MAX_CAP = 1024
SWEEP_CAP = 32          # fused Pauli-string sweep (bmps_pauli_sweep) up to this bond capacity
_RECORD = _native.RECORD_BYTES
RECORD_DTYPE = np.dtype([("err", "<f8"), ("dl", "<i4"), ("dm", "<i4"), ("dr", "<i4"),
                         ("keep", "<i4"), ("status", "<i4"), ("site", "<i4"),
                         ("margin", "<f8"), ("gap", "<f8")])
assert RECORD_DTYPE.itemsize == _RECORD
_ZERO2 = np.zeros((2, 2), dtype=np.complex128)


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _on_device(fn):
    """Run a method with its batch's device current, so the library's launches
    (which use the current device and stream) and the tensors agree."""
    import functools

    @functools.wraps(fn)
    def wrapper(self, *a, **k):
        with torch.cuda.device(self.device):
            return fn(self, *a, **k)
    return wrapper


def require_cuda(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1807_07914_b200 needs a CUDA device (sm_100a); there is no CPU fallback")
    _native.load()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if dev.type != "cuda":
        raise RuntimeError(f"device {dev} is not a CUDA device; there is no CPU fallback")
    return dev


# ---------------------------------------------------------------------------
# lowering and scheduling
# ---------------------------------------------------------------------------

_SWAP = np.ascontiguousarray(SWAP_MATRIX)


def lower_program(program, n: int, validate_matrices: bool = True):
    """Flatten a program into (arity, site, matrix) ops in reference order.

    Non-adjacent two-qubit gates expand into the reference's SWAP chain
    (``mps.py:148-157``); MEASURE is skipped (``backends.py:53-54``). Returns
    arity (int8), site (int32) and a list of matrices.
    """
    arity: list[int] = []
    site: list[int] = []
    mats: list[np.ndarray] = []
    for op in program:
        kind = getattr(op, "kind", None)
        if kind is not None and kind.value == "MEASURE":
            continue
        qs = op.qubits
        for q in qs:
            if not 0 <= q < n:
                raise ValueError(f"site {q} out of range for {n} qubits")
        m = gate_matrix(op)
        if validate_matrices and kind is None:
            check_unitary(m)
        if len(qs) == 1:
            arity.append(1)
            site.append(qs[0])
            mats.append(m)
            continue
        q1, q2 = qs
        if q1 == q2:
            raise ValueError("two-qubit gate needs two distinct sites")
        lo, hi = (q1, q2) if q1 < q2 else (q2, q1)
        for k in range(hi - 1, lo, -1):
            arity.append(2); site.append(k); mats.append(_SWAP)
        arity.append(2); site.append(lo); mats.append(m if q1 < q2 else _SWAP @ m @ _SWAP)
        for k in range(lo + 1, hi):
            arity.append(2); site.append(k); mats.append(_SWAP)
    return np.asarray(arity, dtype=np.int8), np.asarray(site, dtype=np.int32), mats


def asap_layers(arity: np.ndarray, site: np.ndarray, n: int) -> np.ndarray:
    """Earliest layer of each op such that ops sharing a site keep program order."""
    last = np.zeros(n + 1, dtype=np.int64)
    layer = np.empty(len(arity), dtype=np.int64)
    for i in range(len(arity)):
        q = int(site[i])
        if arity[i] == 1:
            L = last[q] + 1
            last[q] = L
        else:
            L = max(last[q], last[q + 1]) + 1
            last[q] = L
            last[q + 1] = L
        layer[i] = L - 1
    return layer


@dataclass
class Plan:
    """A batch of lowered programs scheduled into layers (host arrays)."""

    n_layers: int
    # per layer offsets into the concatenated arrays
    off1: np.ndarray
    off2: np.ndarray
    items1: np.ndarray      # int32 [K1, 2]
    gates1: np.ndarray      # complex128 [K1, 2, 2]
    items2: np.ndarray      # int32 [K2, 2]
    gates2: np.ndarray      # complex128 [K2, 4, 4]
    logidx2: np.ndarray     # int32 [K2]
    ranges: np.ndarray      # int32 [R, 3] (state, first record, count), program order
    n_records: int
    max_state: int = -1     # largest state index the plan touches


_FIXED_1Q = ("I", "X", "Y", "Z", "H")
_FIXED_2Q = ("CNOT", "CZ", "SWAP")
_ROT_NAMES = ("RX", "RY", "RZ")
_CODE_OF = {name: i for i, name in enumerate(_FIXED_1Q + _FIXED_2Q + _ROT_NAMES)}
_CUSTOM = -1
_FIXED_TABLE_1Q = np.stack([gate_matrix(type("G", (), {"kind": type("K", (), {"value": nm})(),
                                                        "params": ()})()) for nm in _FIXED_1Q])
_FIXED_TABLE_2Q = np.stack([gate_matrix(type("G", (), {"kind": type("K", (), {"value": nm})(),
                                                        "params": ()})()) for nm in _FIXED_2Q])
_P4 = [0, 2, 1, 3]
_KINFO: dict = {}


def _kind_info(kind):
    """(code, is_rotation) of a gate kind, None for MEASURE (any enum with the
    reference's string values -- the reference's own ``GateKind`` works)."""
    try:
        return _KINFO[kind]
    except (KeyError, TypeError):
        pass
    name = kind.value
    if name == "MEASURE":
        info = None
    elif name in _CODE_OF:
        info = (_CODE_OF[name], name in _ROT_NAMES)
    else:
        raise ValueError(f"{name} has no unitary matrix")
    try:
        _KINFO[kind] = info
    except TypeError:
        pass
    return info


_UNIFORM_FAST = True


def _extract_uniform(programs):
    """``_extract`` for a batch whose programs all have the first one's structure (same
    gate kinds on the same qubits, op for op -- a VQE ansatz bound to many parameter
    vectors, config 2): the structure is extracted once and tiled, only the rotation
    angles are read per program. None if the batch is not uniform (or has matrix gates)."""
    ref = programs[0]
    try:
        sig = [(op.kind, op.qubits) for op in ref]
        for prog in programs[1:]:
            if len(prog) != len(ref) or [(op.kind, op.qubits) for op in prog] != sig:
                return None
    except AttributeError:          # MatrixGate ops carry no kind
        return None
    # source positions of the kept ops (MEASUREs dropped) and of the rotations among them
    infos = [_kind_info(k) for k, _ in sig]
    kept = [i for i, info in enumerate(infos) if info is not None]
    rot = [j for j, i in enumerate(kept) if infos[i][1]]
    rot_src = [kept[j] for j in rot]
    ar0, q10, q20, code0, _, _, _ = _extract_slow([ref])
    S, m = len(programs), len(kept)
    th = np.zeros((S, m), np.float64)
    if rot:
        th[:, rot] = [[float(prog[i].params[0]) for i in rot_src] for prog in programs]
    return (np.tile(ar0, S), np.tile(q10, S), np.tile(q20, S), np.tile(code0, S),
            th.reshape(-1).tolist(), {}, np.arange(S + 1, dtype=np.int64) * m)


def _extract_slow(programs):
    global _UNIFORM_FAST
    saved, _UNIFORM_FAST = _UNIFORM_FAST, False
    try:
        return _extract(programs)
    finally:
        _UNIFORM_FAST = saved


def _extract(programs):
    """Flat per-op arrays of a batch of programs (MEASUREs dropped): arity, q1,
    q2, gate code, rotation angle, custom matrices by op index, program offsets.
    This loop is the one per-op Python cost of planning (kind lookups cached by
    object identity; enum hashing is slow)."""
    if _UNIFORM_FAST and len(programs) >= 4:
        fast = _extract_uniform(programs)
        if fast is not None:
            return fast
    ar, q1, q2, code, theta = [], [], [], [], []
    ar_a, q1_a, q2_a, code_a, th_a = ar.append, q1.append, q2.append, code.append, theta.append
    custom = {}
    off = [0]
    cache = {}
    for prog in programs:
        for op in prog:
            k = getattr(op, "kind", None)
            e = cache.get(id(k))
            if e is None or e[0] is not k:
                e = (k, None if k is None else _kind_info(k))
                cache[id(k)] = e
            info = e[1]
            if k is None:
                custom[len(ar)] = np.asarray(op.matrix, dtype=np.complex128)
                code_a(_CUSTOM)
                th_a(0.0)
            elif info is None:
                continue
            else:
                code_a(info[0])
                th_a(float(op.params[0]) if info[1] else 0.0)
            qs = op.qubits
            if len(qs) == 1:
                ar_a(1)
                q1_a(qs[0])
                q2_a(qs[0])
            else:
                ar_a(2)
                q1_a(qs[0])
                q2_a(qs[1])
        off.append(len(ar))
    return (np.asarray(ar, np.int8), np.asarray(q1, np.int32), np.asarray(q2, np.int32),
            np.asarray(code, np.int32), theta, custom, np.asarray(off, np.int64))


def _source_matrices(sel: np.ndarray, code: np.ndarray, theta: list, custom: dict, dim: int,
                     validate: bool) -> np.ndarray:
    """Matrices of source ops ``sel`` (all of arity log2(dim)), same bits as gates.py."""
    out = np.empty((len(sel), dim, dim), np.complex128)
    c = code[sel]
    table = _FIXED_TABLE_1Q if dim == 2 else _FIXED_TABLE_2Q
    base = 0 if dim == 2 else len(_FIXED_1Q)
    fixed = (c >= base) & (c < base + len(table))
    out[fixed] = table[c[fixed] - base]
    if dim == 2:
        rot0 = len(_FIXED_1Q) + len(_FIXED_2Q)
        for r, name in enumerate(_ROT_NAMES):
            w = np.nonzero(c == rot0 + r)[0]
            if not len(w):
                continue
            th = [theta[int(i)] for i in sel[w]]
            if name == "RZ":
                t = np.asarray(th)
                blk = np.zeros((len(w), 2, 2), np.complex128)
                blk[:, 0, 0] = np.exp(-1j * t / 2)
                blk[:, 1, 1] = np.exp(1j * t / 2)
            else:
                cs = np.array([cos(x / 2) for x in th])
                sn = np.array([sin(x / 2) for x in th])
                blk = np.empty((len(w), 2, 2), np.complex128)
                blk[:, 0, 0] = cs
                blk[:, 1, 1] = cs
                if name == "RX":
                    off = (-0.0 * sn) + 1j * 0.0
                    off.imag = -1.0 * sn
                    blk[:, 0, 1] = off
                    blk[:, 1, 0] = off
                else:
                    blk[:, 0, 1] = -sn
                    blk[:, 1, 0] = sn
            out[w] = blk
    for j in np.nonzero(c == _CUSTOM)[0]:
        m = custom[int(sel[j])]
        if m.shape != (dim, dim):
            raise ValueError(f"expected a {dim}x{dim} matrix, got shape {m.shape}")
        if validate:
            check_unitary(m)
        out[j] = m
    return out


def compile_batch(programs, n: int, states=None, validate_matrices: bool = True) -> Plan:
    """Lower and layer ``programs[i]`` for state ``states[i]`` (default i).

    Same plan as lowering each program with ``lower_program`` (reference gate
    order and SWAP routing) and layering it with ``asap_layers``; the routing
    and layering run in the native planner (``bmps_plan_build``) and the gate
    matrices are built vectorised, so batches of 10^3 circuits plan in well
    under a second.
    """
    programs = list(programs)
    states = np.arange(len(programs), dtype=np.int32) if states is None else \
        np.asarray(list(states), dtype=np.int32)
    if len(states) != len(programs):
        raise ValueError(f"{len(programs)} programs but {len(states)} state indices")
    if len(states) and (states.min() < 0 or len(np.unique(states)) != len(states)):
        # one program per state per plan: the layering and the in-order stats replay
        # assume a state's ops come from a single program
        raise ValueError("state indices of a plan must be distinct and non-negative")
    ar, q1, q2, code, theta, custom, off = _extract(programs)
    lib = _native.load()
    nx = int(lib.bmps_plan_expanded_count(ar.ctypes.data, q1.ctypes.data, q2.ctypes.data, len(ar)))
    x_state = np.empty(nx, np.int32)
    x_ar = np.empty(nx, np.int8)
    x_site = np.empty(nx, np.int32)
    x_src = np.empty(nx, np.int64)
    x_layer = np.empty(nx, np.int32)
    x_rec = np.empty(nx, np.int64)
    err = ctypes.c_int64(-1)
    rc = lib.bmps_plan_build(len(programs), off.ctypes.data, states.ctypes.data, ar.ctypes.data,
                             q1.ctypes.data, q2.ctypes.data, n, x_state.ctypes.data, x_ar.ctypes.data,
                             x_site.ctypes.data, x_src.ctypes.data, x_layer.ctypes.data,
                             x_rec.ctypes.data, ctypes.byref(err))
    if rc == _native.BMPS_PLAN_E_SITE:
        i = int(err.value)
        bad = next(q for q in ((q1[i],) if ar[i] == 1 else (q1[i], q2[i])) if not 0 <= q < n)
        raise ValueError(f"site {int(bad)} out of range for {n} qubits")
    if rc == _native.BMPS_PLAN_E_SAME_SITE:
        raise ValueError("two-qubit gate needs two distinct sites")
    _native.check(rc, "bmps_plan_build")
    # per-program record ranges (state, first record, count) in program order: a
    # two-qubit source op at distance d expands to 2d - 1 records (SWAP routing)
    w = np.where(ar == 2, 2 * np.abs(q1.astype(np.int64) - q2) - 1, 0)
    cs = np.concatenate([[0], np.cumsum(w)])
    first, counts = cs[off[:-1]], cs[off[1:]] - cs[off[:-1]]
    n_records = int(cs[-1])
    ranges = [(int(states[p]), int(first[p]), int(counts[p])) for p in np.nonzero(counts)[0]]
    max_state = int(states.max()) if len(states) else -1
    if nx == 0:
        return Plan(0, np.zeros(1, np.int64), np.zeros(1, np.int64), np.zeros((0, 2), np.int32),
                    np.zeros((0, 2, 2), complex), np.zeros((0, 2), np.int32),
                    np.zeros((0, 4, 4), complex), np.zeros(0, np.int32),
                    np.zeros((0, 3), np.int32), 0, max_state)
    n_layers = int(x_layer.max()) + 1
    # stable order: layer, then original (state-major, program) order
    order = np.argsort(x_layer, kind="stable")
    one = order[x_ar[order] == 1]
    two = order[x_ar[order] == 2]
    items1 = np.stack([x_state[one], x_site[one]], axis=1).astype(np.int32)
    items2 = np.stack([x_state[two], x_site[two]], axis=1).astype(np.int32)
    # gate tables
    src1 = np.nonzero(ar == 1)[0]
    src2 = np.nonzero(ar == 2)[0]
    pos = np.full(len(ar), -1, np.int64)
    pos[src1] = np.arange(len(src1))
    pos[src2] = np.arange(len(src2))
    m1 = _source_matrices(src1, code, theta, custom, 2, validate_matrices)
    m2 = _source_matrices(src2, code, theta, custom, 4, validate_matrices)
    gates1 = m1[pos[x_src[one]]] if len(one) else np.zeros((0, 2, 2), np.complex128)
    s2 = x_src[two]
    direct, swapped = s2 >= 0, s2 <= -2
    gates2 = np.empty((len(two), 4, 4), np.complex128)
    gates2[s2 == -1] = _SWAP
    if direct.any():
        gates2[direct] = m2[pos[s2[direct]]]
    if swapped.any():
        g = m2[pos[-s2[swapped] - 2]]
        gates2[swapped] = g[:, _P4][:, :, _P4]       # SWAP . G . SWAP (mps.py:154)
    lay_one, lay_two = x_layer[one], x_layer[two]
    off1 = np.searchsorted(lay_one, np.arange(n_layers + 1)) if len(one) else np.zeros(n_layers + 1, np.int64)
    off2 = np.searchsorted(lay_two, np.arange(n_layers + 1)) if len(two) else np.zeros(n_layers + 1, np.int64)
    return Plan(n_layers, off1, off2, items1, gates1, items2, gates2, x_rec[two].astype(np.int32),
                np.asarray(ranges, dtype=np.int32).reshape(-1, 3), n_records, max_state)


# ---------------------------------------------------------------------------
# device state batch
# ---------------------------------------------------------------------------


class SvdTimer:
    """CUDA-event pairs the library records around the SVD stage (column sort, QR
    preconditioner, Jacobi, double-QR epilogue) of every ``bmps_apply_2q`` call of
    the batches it is attached to (``bmps_params.svd_events``), on the launching
    stream. Bench instrumentation; ``total_ms`` synchronises."""

    def __init__(self, capacity: int = 4096):
        self.capacity = int(capacity)
        self.events = []
        for _ in range(2 * self.capacity):
            e = torch.cuda.Event(enable_timing=True)
            e.record()                     # creates the underlying cudaEvent_t
            self.events.append(e)
        self.handles = (ctypes.c_void_p * (2 * self.capacity))(*[e.cuda_event for e in self.events])
        self.used = ctypes.c_int32(0)
        torch.cuda.synchronize()

    def attach(self, batch: "MpsBatch") -> None:
        batch.svd_timer = (self.handles, self.used, self.capacity)

    def reset(self) -> None:
        self.used.value = 0

    def total_ms(self) -> tuple[float, int]:
        n = self.used.value
        tot = 0.0
        for i in range(n):
            self.events[2 * i + 1].synchronize()
            tot += self.events[2 * i].elapsed_time(self.events[2 * i + 1])
        return tot, n


class _DevPtr:
    """A raw device address with the ``data_ptr()`` of a tensor view."""

    __slots__ = ("p",)

    def __init__(self, p: int):
        self.p = p

    def data_ptr(self) -> int:
        return self.p


class _Staging:
    """Ring of pinned host / device argument slots for per-gate launches. A slot
    is reused only after the event recorded behind its H2D copy has completed,
    so a host write can never race an in-flight copy."""

    SLOT = 512   # bytes: item (8) | log index (4) | range (12) | ... | gate at 64 (256)

    def __init__(self, device, slots: int = 64):
        self.n = slots
        self.host = torch.empty(slots * self.SLOT, dtype=torch.uint8).pin_memory()
        self.host_i32 = self.host.numpy().view(np.int32)
        self.dev = torch.empty(slots * self.SLOT, dtype=torch.uint8, device=device)
        self.events = [None] * slots
        self.k = 0

    def acquire(self):
        slot = self.k % self.n
        self.k += 1
        ev = self.events[slot]
        if ev is not None:
            ev.synchronize()
        w = self.SLOT // 4
        return self.host_i32[slot * w:(slot + 1) * w], self.dev.data_ptr() + slot * self.SLOT, slot

    def commit(self, slot: int, nbytes: int) -> None:
        a = slot * self.SLOT
        self.dev[a:a + nbytes].copy_(self.host[a:a + nbytes], non_blocking=True)
        ev = self.events[slot] or torch.cuda.Event()
        ev.record()
        self.events[slot] = ev


class GraphedPlan:
    """A plan run from |0...0> as ONE CUDA-graph launch: ``batch.reset()`` followed by
    every layer of ``plan`` (the per-gate loop of
    ``backends.py:52-59`` captured instead of re-issued).

    For launch-bound work that repeats the same circuit STRUCTURE with new gate
    matrices -- a VQE optimiser re-evaluating an ansatz at new angles (config 2: 76
    sequential CNOT-ladder layers of tiny kernels, ~800 launches per evaluation) --
    ``replay(gates1, gates2)`` copies the new matrices into the captured buffers and
    launches the graph: no per-layer Python, ctypes or launch overhead. The first
    construction runs the plan once eagerly (that sizes the bond capacity and the
    workspace, which a graph cannot do), then records the second run. Results are
    those of ``reset(); execute(plan)`` bit for bit (same kernels, same order).

    The graph holds raw device pointers: it keeps its workspace alive itself, and
    ``replay`` refuses to run if the batch has re-allocated its state tensors since
    (a later plan that grew the bond capacity) -- capture again in that case.
    """

    def __init__(self, batch: "MpsBatch", plan: Plan, mode: int = 0):
        if plan.n_layers == 0:
            raise ValueError("empty plan")
        if plan.max_state >= batch.S:
            raise ValueError(f"plan addresses state {plan.max_state}, batch has {batch.S}")
        self.batch, self.plan, self.mode = batch, plan, mode
        with torch.cuda.device(batch.device):
            # capacity by the host's bound model, not the warm run's true bonds: replays
            # with other matrices may need more than this run did, and the recorded run
            # must not ask the device (a sync) -- so no refresh_bounds here
            batch._by_model = True
            try:
                self._record(batch, plan, mode)
            finally:
                batch._by_model = False
        if batch._ws is not self._ws or batch.gamma is not self._state[0]:
            raise RuntimeError("capacity or workspace changed during capture")

    def _record(self, batch, plan, mode) -> None:
        batch.reset()
        batch.execute(plan, mode)            # sizes capacity + workspace, first-use setup
        torch.cuda.synchronize()
        batch.check_status()
        self._bufs = batch._upload(plan)
        self._log = torch.empty(max(plan.n_records, 1) * _RECORD, dtype=torch.uint8,
                                device=batch.device)
        torch.cuda.synchronize()
        self._state = (batch.gamma, batch.lam, batch.dims)
        self._ws = batch._ws                 # stays alive with the graph
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            batch.reset()
            batch._launch(plan, self._bufs, self._log, mode)
        self._dim_ub = batch.dim_ub.copy()

    def replay(self, gates1=None, gates2=None) -> "MpsBatch":
        """Run the captured plan again from |0...0> (asynchronous). ``gates1`` [n1, 2, 2]
        / ``gates2`` [n2, 4, 4] complex128 replace the plan's matrices in plan order
        (``Plan.gates1`` / ``Plan.gates2`` of a plan compiled from the re-bound programs)."""
        b = self.batch
        if b.gamma is not self._state[0] or b.lam is not self._state[1] or b.dims is not self._state[2]:
            raise RuntimeError("the batch re-allocated its state since capture; capture the plan again")
        with torch.cuda.device(b.device):
            hosts = self._bufs[6]
            for new, dev_t, host_t in ((gates1, self._bufs[1], hosts[1]), (gates2, self._bufs[3], hosts[3])):
                if new is None:
                    continue
                a = np.ascontiguousarray(new, dtype=np.complex128).view(np.float64).reshape(-1)
                if a.size != host_t.numel():
                    raise ValueError(f"the captured plan holds {host_t.numel()} doubles of gate "
                                     f"matrices here, got {a.size}")
                # the previous replay's copy out of this pinned buffer must be done
                torch.cuda.current_stream().synchronize()
                host_t.view(-1).numpy()[:] = a
                dev_t.view(-1).copy_(host_t.view(-1), non_blocking=True)
            self.graph.replay()
        b.dim_ub[:] = self._dim_ub
        entry = (self._log, self.plan.ranges)
        b._logs = b._logs + [entry] if b.keep_records else [entry]
        return b


class MpsBatch:
    """S independent n-qubit MPS states resident in HBM, initially |0...0>.

    ``keep_records`` retains every executed plan's per-update records on the
    device (for ``update_records``); by default only the most recent plan's are
    kept, so a long per-gate loop does not grow device memory. Per-bond
    truncation, the cutoff-tie margin and the truncation gap are accumulated on
    the device for every update regardless.
    """

    def __init__(self, num_states: int, n: int, policy: TruncationPolicy | None = None,
                 device=None, cap: int | None = None, max_items_per_launch: int = 4096,
                 workspace_budget: int = 24 << 30, keep_records: bool = False):
        if n < 1:
            raise ValueError("need at least one qubit")
        if num_states < 1:
            raise ValueError("need at least one state")
        self.device = require_cuda(device)
        self.lib = _native.load()
        self.S = int(num_states)
        self.n = int(n)
        self.policy = policy or TruncationPolicy()
        self.max_items = int(max_items_per_launch)
        self.workspace_budget = int(workspace_budget)
        self.keep_records = bool(keep_records)
        self.cap = 1
        self.dim_ub = np.ones((self.S, self.n + 1), dtype=np.int64)
        self._ws = None
        self._ws_bytes = 0
        self._logs: list = []
        self.svd_timer = None       # bench hook: (events array, used counter, capacity)
        self._by_model = False      # size capacity by the host bound model only (graph capture)
        with torch.cuda.device(self.device):
            self._alloc(int(cap) if cap else 1)
            self.reset()

    # -- buffers ---------------------------------------------------------------
    def _alloc(self, cap: int) -> None:
        S, n, dev = self.S, self.n, self.device
        self.cap = cap
        self.gamma = torch.zeros((S, n, cap, 2, cap), dtype=torch.complex128, device=dev)
        self.lam = torch.zeros((S, n + 1, cap), dtype=torch.float64, device=dev)
        self.dims = torch.ones((S, n + 1), dtype=torch.int32, device=dev)
        if not hasattr(self, "trunc_err"):
            self.trunc_err = torch.zeros(S, dtype=torch.float64, device=dev)
            self.entries = torch.zeros(S, dtype=torch.int64, device=dev)
            self.peak = torch.zeros(S, dtype=torch.int64, device=dev)
            self.mbs = torch.zeros(S, dtype=torch.int32, device=dev)
            self.status = torch.zeros(S, dtype=torch.int32, device=dev)
            self.status_bond = torch.zeros(S, dtype=torch.int32, device=dev)
            self.bond_err = torch.zeros((S, max(n - 1, 1)), dtype=torch.float64, device=dev)
            self.min_margin = torch.full((S,), float("inf"), dtype=torch.float64, device=dev)
            self.min_gap = torch.full((S,), float("inf"), dtype=torch.float64, device=dev)

    @_on_device
    def reset(self) -> None:
        """Re-initialise every state to |0...0> (``mps.py:55-66``)."""
        self.gamma.zero_()
        self.lam.zero_()
        self.dim_ub[:] = 1
        self._logs = []
        self.bond_err.zero_()
        self.min_margin.fill_(float("inf"))
        self.min_gap.fill_(float("inf"))
        rc = self.lib.bmps_init_product(
            _ptr(self.gamma), _ptr(self.lam), _ptr(self.dims), _ptr(self.trunc_err),
            _ptr(self.entries), _ptr(self.peak), _ptr(self.mbs), _ptr(self.status),
            _ptr(self.status_bond), self.S, self.n, self.cap, _stream())
        _native.check(rc, "bmps_init_product")

    def _cap_limit(self) -> int:
        full = 1 << min(self.n // 2, 30)
        mb = self.policy.max_bond
        return min(full, mb) if mb is not None else full

    @_on_device
    def ensure_capacity(self, needed: int) -> None:
        """Grow the bond capacity (power of two) to hold ``needed``; copies state."""
        if needed <= self.cap:
            return
        if needed > MAX_CAP:
            raise ValueError(
                f"bond dimension {needed} exceeds the device capacity limit {MAX_CAP}; "
                "set TruncationPolicy.max_bond")
        new = 1
        while new < needed:
            new <<= 1
        new = min(new, max(MAX_CAP, needed))
        old_g, old_l, old_d, oc = self.gamma, self.lam, self.dims, self.cap
        self._alloc(new)
        self.gamma[:, :, :oc, :, :oc] = old_g
        self.lam[:, :, :oc] = old_l
        self.dims.copy_(old_d)

    def refresh_bounds(self) -> None:
        """Replace the host's upper-bound model of the bond dims by the true dims
        (one device sync). Called before the model would force a capacity growth,
        so growth and the capacity limit follow the real bonds, not the bound --
        e.g. CNOT layers on |0...0> keep every bond at 1 however deep they go."""
        self.dim_ub[:] = self.dims.cpu().numpy()

    def _workspace(self, nitems: int) -> tuple[int, int]:
        need = int(self.lib.bmps_apply_2q_workspace_bytes(self.cap, nitems))
        if self._ws is None or self._ws_bytes < need:
            self._ws = torch.empty(need, dtype=torch.uint8, device=self.device)
            self._ws_bytes = need
        return self._ws.data_ptr(), self._ws_bytes

    def _params(self, mode: int = 0):
        extra = {"jacobi_mode": mode} if mode else {}
        p = _native.params(**extra)
        t = self.svd_timer
        if t is not None:
            p.svd_events = ctypes.cast(t[0], ctypes.c_void_p)
            p.svd_events_used = ctypes.cast(ctypes.pointer(t[1]), ctypes.c_void_p)
            p.n_svd_events = t[2]
        return p

    # -- execution ---------------------------------------------------------------
    def run(self, programs, states=None, mode: int = 0) -> "MpsBatch":
        """Apply ``programs[i]`` to state ``states[i]`` (default: i)."""
        plan = compile_batch(programs, self.n, states)
        self.execute(plan, mode=mode)
        return self

    @_on_device
    def execute(self, plan: Plan, mode: int = 0) -> None:
        """Launch a plan layer by layer (asynchronous; no host sync unless the bond
        bound model asks for more capacity than allocated)."""
        if plan.n_layers == 0:
            return
        if plan.max_state >= self.S:
            raise ValueError(f"plan addresses state {plan.max_state}, batch has {self.S}")
        bufs = self._upload(plan)
        log = torch.empty(max(plan.n_records, 1) * _RECORD, dtype=torch.uint8, device=self.device)
        self._launch(plan, bufs, log, mode)
        self._keep_alive = bufs

    def _upload(self, plan: Plan) -> tuple:
        """The plan's item / gate / log-index / range arrays on the device (pinned
        staging, asynchronous copies): (it1, g1, it2, g2, li2, rng, pinned hosts)."""
        dev = self.device
        hosts = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
                 for a in (plan.items1, plan.gates1.view(np.float64), plan.items2,
                           plan.gates2.view(np.float64), plan.logidx2, plan.ranges)]
        return tuple(h.to(dev, non_blocking=True) for h in hosts) + (hosts,)

    def _launch(self, plan: Plan, bufs: tuple, log: torch.Tensor, mode: int = 0) -> None:
        """Every layer's launches on the current stream (stream-ordered work only once
        the capacity and workspace are sized: what ``capture`` records into a graph)."""
        it1, g1, it2, g2, li2, rng = bufs[:6]
        pol = self.policy.as_c()
        params = self._params(mode)
        lim = self._cap_limit()
        stream = _stream()
        for L in range(plan.n_layers):
            a, b = int(plan.off1[L]), int(plan.off1[L + 1])
            if b > a:
                rc = self.lib.bmps_apply_1q(
                    _ptr(self.gamma), _ptr(self.dims), self.S, self.n, self.cap,
                    it1.data_ptr() + 8 * a, g1.data_ptr() + 64 * a, b - a, stream)
                _native.check(rc, "bmps_apply_1q")
            a, b = int(plan.off2[L]), int(plan.off2[L + 1])
            if b <= a:
                continue
            self._apply_2q_layer(plan.items2[a:b], it2, g2, li2, a, b, log, pol, params, lim, stream)
        self._replay(log, rng, len(plan.ranges), stream)
        if self.keep_records:
            self._logs.append((log, plan.ranges))
        else:
            self._logs = [(log, plan.ranges)]

    def capture(self, plan: Plan, mode: int = 0) -> "GraphedPlan":
        """``reset()`` + ``execute(plan)`` recorded once into a CUDA graph that can be
        replayed with new gate matrices (see ``GraphedPlan``)."""
        return GraphedPlan(self, plan, mode)

    def _apply_2q_layer(self, its, it2, g2, li2, a, b, log, pol, params, lim, stream) -> None:
        s_idx, q = its[:, 0], its[:, 1]
        ub = self.dim_ub
        need = lambda: int(max(ub[s_idx, q].max(), ub[s_idx, q + 2].max(),
                               np.minimum(np.minimum(2 * ub[s_idx, q], 2 * ub[s_idx, q + 2]), lim).max()))
        if need() > self.cap and not self._by_model:
            self.refresh_bounds()      # the bound model may overestimate: consult the device
        self.ensure_capacity(need())
        bound = int(max(ub[s_idx, q].max(), ub[s_idx, q + 2].max()))
        new = np.minimum(np.minimum(2 * ub[s_idx, q], 2 * ub[s_idx, q + 2]), lim)
        per_item = int(self.lib.bmps_apply_2q_workspace_bytes(self.cap, 1))
        chunk = max(1, min(self.max_items, self.workspace_budget // max(per_item, 1)))
        # visits of one Jacobi round, from the per-item bounds: columns = 2 min(dl, dr),
        # blocks of 16 paired up (bmps_params.visits_hint)
        blocks = (2 * np.minimum(ub[s_idx, q], ub[s_idx, q + 2]) + 15) // 16
        visits = np.maximum(1, (blocks + (blocks & 1)) // 2)
        for c0 in range(a, b, chunk):
            c1 = min(b, c0 + chunk)
            ws, wsb = self._workspace(c1 - c0)
            params.visits_hint = int(min(visits[c0 - a:c1 - a].sum(), 2 ** 31 - 1))
            rc = self.lib.bmps_apply_2q(
                _ptr(self.gamma), _ptr(self.lam), _ptr(self.dims), self.S, self.n, self.cap,
                it2.data_ptr() + 8 * c0, g2.data_ptr() + 256 * c0, c1 - c0, pol,
                log.data_ptr(), li2.data_ptr() + 4 * c0, ws, wsb, min(bound, self.cap),
                ctypes.byref(params), stream)
            _native.check(rc, "bmps_apply_2q")
        ub[s_idx, q + 1] = new

    def _replay(self, log, rng, nranges, stream) -> None:
        rc = self.lib.bmps_stats_replay(
            log.data_ptr(), rng.data_ptr(), nranges, _ptr(self.trunc_err), _ptr(self.entries),
            _ptr(self.peak), _ptr(self.mbs), _ptr(self.status), _ptr(self.status_bond),
            _ptr(self.bond_err) if self.n > 1 else None, self.n, _ptr(self.min_margin),
            _ptr(self.min_gap), stream)
        _native.check(rc, "bmps_stats_replay")

    # -- per-gate path (the reference's own callers loop gate by gate) -----------
    @_on_device
    def apply_ops(self, s: int, ops) -> None:
        """Apply (arity, site, matrix) ops to state ``s`` in order, one op per layer,
        without the planner: the drop-in ``MpsState.apply_*`` path. Arguments go
        through a ring of pinned staging slots (no host allocation per gate) and
        the launches stay asynchronous."""
        if not 0 <= s < self.S:
            raise ValueError(f"state {s} out of range for {self.S} states")
        st = getattr(self, "_staging", None)
        if st is None:
            st = self._staging = _Staging(self.device)
        stream = _stream()
        pol = None
        params = None
        lim = self._cap_limit()
        for arity, site, mat in ops:
            h, d, slot = st.acquire()
            m = np.ascontiguousarray(mat, dtype=np.complex128)
            h[0:2] = (s, site)
            if arity == 1:
                h.view(np.complex128)[4:8] = m.reshape(-1)
                st.commit(slot, 128)
                rc = self.lib.bmps_apply_1q(_ptr(self.gamma), _ptr(self.dims), self.S, self.n, self.cap,
                                            d, d + 64, 1, stream)
                _native.check(rc, "bmps_apply_1q")
                continue
            if pol is None:
                pol, params = self.policy.as_c(), self._params()
            h[4] = 0                      # log index
            h[8:11] = (s, 0, 1)           # replay range (state, first record, count)
            h.view(np.complex128)[4:20] = m.reshape(-1)
            st.commit(slot, 320)
            log = torch.empty(_RECORD, dtype=torch.uint8, device=self.device)
            its = np.array([[s, site]], np.int32)
            self._apply_2q_layer(its, _DevPtr(d), _DevPtr(d + 64), _DevPtr(d + 16), 0, 1, log,
                                 pol, params, lim, stream)
            self._replay(log, _DevPtr(d + 32), 1, stream)
            if self.keep_records:
                self._logs.append((log, np.array([[s, 0, 1]], np.int32)))
            else:
                self._logs = [(log, np.array([[s, 0, 1]], np.int32))]

    @_on_device
    def last_sweeps(self, count: int | None = None) -> np.ndarray:
        """Jacobi sweeps of the items of the most recent bmps_apply_2q launch."""
        if self._ws is None:
            return np.zeros(0, np.int32)
        n = count if count is not None else self.max_items
        out = torch.zeros(n, dtype=torch.int32, device=self.device)
        rc = self.lib.bmps_apply_2q_sweeps(self._ws.data_ptr(), n, out.data_ptr(), _stream())
        _native.check(rc, "bmps_apply_2q_sweeps")
        return out.cpu().numpy()

    def update_records(self, s: int) -> np.ndarray:
        """Per-update records of state ``s`` in program order (the retained plans:
        all of them with ``keep_records``, else the most recent)."""
        out = []
        for log, ranges in self._logs:
            rec = log.cpu().numpy().view(RECORD_DTYPE)
            for st, first, cnt in ranges:
                if st == s:
                    out.append(rec[first:first + cnt])
        return np.concatenate(out) if out else np.zeros(0, RECORD_DTYPE)

    def bond_truncation(self, s: int = 0) -> np.ndarray:
        """Discarded weight per bond since the last reset (reference bond index q =
        site of the update), accumulated on the device in program order."""
        self.check_status()
        if self.n < 2:
            return np.zeros(0)
        return self.bond_err[s].cpu().numpy()

    def decision_margins(self) -> tuple[np.ndarray, np.ndarray]:
        """Per state, the smallest cutoff-tie margin and truncation gap over all
        updates since the last reset (``bmps_update_record.margin`` / ``gap``)."""
        return self.min_margin.cpu().numpy(), self.min_gap.cpu().numpy()

    # -- status and host views ---------------------------------------------------
    def check_status(self) -> None:
        """Raise the reference's RuntimeError for the first failed state (syncs)."""
        st = self.status.cpu().numpy()
        bad = np.nonzero(st)[0]
        if len(bad) == 0:
            return
        s = int(bad[0])
        code = int(st[s])
        q = int(self.status_bond[s].item())
        if code == _native.BMPS_S_SVD_FAILED:
            raise RuntimeError(f"SVD failed on bond {q}")
        if code == _native.BMPS_S_ALL_TRUNCATED:
            raise RuntimeError(f"all singular values truncated on bond {q}")
        raise RuntimeError(f"state {s}: {self.lib.bmps_status_string(code).decode()} (bond {q})")

    def host_dims(self) -> np.ndarray:
        return self.dims.cpu().numpy()

    def site_tensors(self, s: int = 0) -> list[np.ndarray]:
        d = self.host_dims()[s]
        g = self.gamma[s].cpu().numpy()
        return [np.ascontiguousarray(g[k, : d[k], :, : d[k + 1]]) for k in range(self.n)]

    def bond_vectors(self, s: int = 0) -> list[np.ndarray]:
        d = self.host_dims()[s]
        lam = self.lam[s].cpu().numpy()
        return [lam[b, : d[b]].copy() for b in range(1, self.n)]

    @_on_device
    def load_state(self, s: int, site_tensors, bond_vectors) -> None:
        """Overwrite state ``s`` with host Gamma/lambda (Vidal form, reference layout)."""
        dims = [1] + [len(v) for v in bond_vectors] + [1]
        self.ensure_capacity(max(dims))
        cap = self.cap
        g = np.zeros((self.n, cap, 2, cap), dtype=np.complex128)
        lam = np.zeros((self.n + 1, cap))
        for k, t in enumerate(site_tensors):
            t = np.asarray(t, dtype=np.complex128)
            assert t.shape == (dims[k], 2, dims[k + 1]), (k, t.shape, dims)
            g[k, : dims[k], :, : dims[k + 1]] = t
        lam[0, 0] = 1.0
        lam[self.n, 0] = 1.0
        for b, v in enumerate(bond_vectors, start=1):
            lam[b, : len(v)] = v
        self.gamma[s].copy_(torch.from_numpy(g))
        self.lam[s].copy_(torch.from_numpy(lam))
        self.dims[s].copy_(torch.tensor(dims, dtype=torch.int32))
        self.dim_ub[s] = dims
        ent = sum(dims[k] * 2 * dims[k + 1] for k in range(self.n))
        self.entries[s] = ent
        self.peak[s] = ent
        self.mbs[s] = max(dims)

    # -- queries -------------------------------------------------------------------
    @_on_device
    def amplitudes(self, state_idx, bitstrings) -> np.ndarray:
        """<bits|psi_s> for each (s, bits) (``mps.py:172-179``)."""
        n = self.n
        bits = np.empty((len(bitstrings), n), dtype=np.uint8)
        for i, b in enumerate(bitstrings):
            if len(b) != n or any(c not in "01" for c in b):
                raise ValueError(f"need a bitstring of length {n}, got {b!r}")
            bits[i] = np.frombuffer(b.encode(), dtype=np.uint8) - ord("0")
        self.check_status()
        sidx = torch.as_tensor(np.asarray(state_idx, dtype=np.int32)).to(self.device)
        dbits = torch.from_numpy(bits).to(self.device)
        out = torch.empty(len(bitstrings), dtype=torch.complex128, device=self.device)
        rc = self.lib.bmps_amplitudes(_ptr(self.gamma), _ptr(self.lam), _ptr(self.dims), self.S, n,
                                      self.cap, sidx.data_ptr(), dbits.data_ptr(), len(bitstrings),
                                      out.data_ptr(), _stream())
        _native.check(rc, "bmps_amplitudes")
        return out.cpu().numpy()

    @_on_device
    def sample_bits(self, s: int, uniforms: np.ndarray) -> np.ndarray:
        """Sampled bitstrings (uint8 [shots, n]) of state ``s`` for pre-drawn uniforms."""
        self.check_status()
        shots = uniforms.shape[0]
        u = torch.from_numpy(np.ascontiguousarray(uniforms, dtype=np.float64)).to(self.device)
        sidx = torch.full((shots,), s, dtype=torch.int32, device=self.device)
        bits = torch.empty((shots, self.n), dtype=torch.uint8, device=self.device)
        rc = self.lib.bmps_sample(_ptr(self.gamma), _ptr(self.lam), _ptr(self.dims), self.S, self.n,
                                  self.cap, sidx.data_ptr(), u.data_ptr(), shots, bits.data_ptr(),
                                  _stream())
        _native.check(rc, "bmps_sample")
        return bits.cpu().numpy()

    @_on_device
    def conditional_prob_zero(self, s: int, prefix_vec, k: int):
        """``MpsState.conditional_prob_zero`` (``mps.py:206-214``) on the device:
        (P(qubit k = 0 | prefix), w0, w1) with w_b = prefix @ T_k[:, b, :]."""
        if not 0 <= k < self.n:
            raise ValueError(f"site {k} out of range for {self.n} qubits")
        self.check_status()
        d = self.host_dims()[s]
        pv = np.asarray(prefix_vec, dtype=np.complex128).reshape(-1)
        if len(pv) != d[k]:
            raise ValueError(f"prefix vector has length {len(pv)}, bond {k} has dimension {d[k]}")
        dev = self.device
        pre = torch.from_numpy(pv.copy()).to(dev)
        w = torch.empty((2, max(int(d[k + 1]), 1)), dtype=torch.complex128, device=dev)
        p01 = torch.empty(2, dtype=torch.float64, device=dev)
        rc = self.lib.bmps_conditional(_ptr(self.gamma), _ptr(self.lam), _ptr(self.dims), self.S,
                                       self.n, self.cap, int(s), int(k), pre.data_ptr(),
                                       w[0].data_ptr(), w[1].data_ptr(), p01.data_ptr(), _stream())
        _native.check(rc, "bmps_conditional")
        p0, p1 = (float(x) for x in p01.cpu().numpy())
        wh = w.cpu().numpy()[:, : int(d[k + 1])]
        total = p0 + p1
        return (p0 / total if total > 0 else 0.5), wh[0].copy(), wh[1].copy()

    def sample(self, s: int, shots: int, rng: np.random.Generator) -> dict[str, int]:
        """Counts of full-register bitstrings (``mps.py:216-237``, same uniform stream)."""
        if shots < 1:
            raise ValueError("shots must be >= 1")
        uniforms = rng.random((shots, self.n))   # one draw per qubit per shot, qubit order
        bits = self.sample_bits(s, uniforms)
        counts: dict[str, int] = {}
        for row in bits:
            key = row.tobytes().translate(bytes.maketrans(b"\x00\x01", b"01")).decode()
            counts[key] = counts.get(key, 0) + 1
        return counts

    def _transfer(self, sidx: torch.Tensor, site: torch.Tensor, codes: torch.Tensor, direction: int,
                  env_in: torch.Tensor, in_stride: int, env_out: torch.Tensor, out_stride: int,
                  count: int, in_idx: torch.Tensor | None = None,
                  out_idx: torch.Tensor | None = None) -> None:
        scratch = self._scratch(count)
        rc = self.lib.bmps_env_transfer(
            _ptr(self.gamma), _ptr(self.lam), _ptr(self.dims), self.S, self.n, self.cap,
            sidx.data_ptr(), site.data_ptr(), codes.data_ptr(), direction, env_in.data_ptr(), in_stride,
            _ptr(in_idx), env_out.data_ptr(), out_stride, _ptr(out_idx), scratch.data_ptr(), count,
            _stream())
        _native.check(rc, "bmps_env_transfer")

    def _scratch(self, count: int) -> torch.Tensor:
        need = 2 * count * 2 * self.cap * self.cap
        buf = getattr(self, "_scr", None)
        if buf is None or buf.numel() < need:
            buf = torch.empty(need, dtype=torch.complex128, device=self.device)
            self._scr = buf
        return buf

    def _env_chunk(self) -> int:
        # bound transfer scratch to ~2 GiB
        return max(1, min(4096, (2 << 30) // (64 * self.cap * self.cap)))

    def _identity_env(self, count: int) -> torch.Tensor:
        e = torch.zeros((count, self.cap, self.cap), dtype=torch.complex128, device=self.device)
        e[:, 0, 0] = 1.0
        return e

    @_on_device
    def environments(self, states: np.ndarray, direction: int) -> torch.Tensor:
        """All identity environments L_k (direction 0) or R_k (1), k = 0..n."""
        ns, n, cap = len(states), self.n, self.cap
        env = torch.zeros((ns, n + 1, cap, cap), dtype=torch.complex128, device=self.device)
        sidx = torch.as_tensor(np.asarray(states, dtype=np.int32)).to(self.device)
        codes = torch.zeros(ns, dtype=torch.uint8, device=self.device)
        stride = (n + 1) * cap * cap
        if direction == 0:
            env[:, 0, 0, 0] = 1.0
            steps = range(n)
        else:
            env[:, n, 0, 0] = 1.0
            steps = range(n - 1, -1, -1)
        if cap <= SWEEP_CAP:
            rc = self.lib.bmps_env_sweep(_ptr(self.gamma), _ptr(self.lam), _ptr(self.dims), self.S, n,
                                         cap, sidx.data_ptr(), ns, direction, env.data_ptr(), stride,
                                         _stream())
            _native.check(rc, "bmps_env_sweep")
            return env
        for k in steps:
            site = torch.full((ns,), k, dtype=torch.int32, device=self.device)
            src, dst = (k, k + 1) if direction == 0 else (k + 1, k)
            for c0 in range(0, ns, self._env_chunk()):
                c1 = min(ns, c0 + self._env_chunk())
                self._transfer(sidx[c0:c1], site[c0:c1], codes[c0:c1], direction,
                               env[c0:, src], stride, env[c0:, dst], stride, c1 - c0)
        return env

    @_on_device
    def expectations(self, state_idx, paulis, use_env: bool | None = None) -> np.ndarray:
        """<psi_s|P|psi_s> for each (s, P), real part; RuntimeError on |Im| > 1e-10.

        Reassociates the reference's left-to-right sweep (``mps.py:196-204``):
        each string is swept from its first to its last non-identity site,
        starting from the cached identity environment L_lo and closed with R_{hi+1}.
        """
        n = self.n
        state_idx = np.asarray(state_idx, dtype=np.int32)
        codes = encode_paulis(paulis, n)
        self.check_status()
        npairs = len(paulis)
        if npairs == 0:
            return np.zeros(0)
        sup = codes != 0
        lo = np.where(sup.any(1), sup.argmax(1), 0).astype(np.int32)
        hi = np.where(sup.any(1), n - 1 - sup[:, ::-1].argmax(1), -1).astype(np.int32)
        uniq, inv = np.unique(state_idx, return_inverse=True)
        if use_env is None:
            use_env = npairs > 2 * len(uniq)
        dev, cap = self.device, self.cap
        if use_env:
            Lenv = self.environments(uniq, 0)
            Renv = self.environments(uniq, 1)
        else:
            lo[:] = 0
            hi[:] = n - 1
        out = np.empty(npairs, dtype=np.complex128)
        if use_env and cap <= SWEEP_CAP:
            # small bonds: every string in one fused sweep launch (bmps_pauli_sweep)
            stride = (n + 1) * cap * cap
            res = torch.empty(npairs, dtype=torch.complex128, device=dev)
            args = [torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in
                    (state_idx, inv.astype(np.int32), codes, lo, hi)]
            rc = self.lib.bmps_pauli_sweep(
                _ptr(self.gamma), _ptr(self.lam), _ptr(self.dims), self.S, n, cap,
                *(a.data_ptr() for a in args), Lenv.data_ptr(), Renv.data_ptr(), stride, npairs,
                res.data_ptr(), _stream())
            _native.check(rc, "bmps_pauli_sweep")
            out[:] = res.cpu().numpy()
            bad = np.abs(out.imag) > 1e-10
            if bad.any():
                raise RuntimeError(f"expectation has imaginary residue {out.imag[bad][0]:.3e}")
            return out.real.copy()
        # cap > 32: each string is swept from its cached left environment L_lo over its
        # support on the DMMA transfer GEMMs, one launch pair per site step for all
        # strings still active, environments addressed through device index arrays
        # (no gathers or scatters), and closed against the cached R_{hi+1}
        E = n + 1
        cc = cap * cap
        to_dev = lambda a, dt=np.int32: torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(dev)
        if use_env:
            Lflat = Lenv.view(len(uniq) * E, cap, cap)
            Rflat = Renv.view(len(uniq) * E, cap, cap)
        else:
            Lflat = Rflat = self._identity_env(1)
        chunk = self._env_chunk()
        for c0 in range(0, npairs, chunk):
            c1 = min(npairs, c0 + chunk)
            cnt = c1 - c0
            lo_c, hi_c = lo[c0:c1], hi[c0:c1]
            u_c = inv[c0:c1] if use_env else np.zeros(cnt, np.int64)
            span = np.where(hi_c >= lo_c, hi_c - lo_c + 1, 0)
            codes_c = codes[c0:c1]
            cur = torch.empty((2, cnt, cap, cap), dtype=torch.complex128, device=dev)
            for t in range(int(span.max()) if cnt else 0):
                act = np.nonzero(span > t)[0]
                if len(act) == 0:
                    break
                site_h = (lo_c[act] + t).astype(np.int32)
                if t == 0:
                    src = Lflat
                    in_idx = u_c[act] * E + lo_c[act] if use_env else np.zeros(len(act))
                else:
                    src, in_idx = cur[(t - 1) & 1], act
                self._transfer(to_dev(state_idx[c0:c1][act]), to_dev(site_h),
                               to_dev(codes_c[act, site_h], np.uint8), 0, src, cc, cur[t & 1], cc,
                               len(act), in_idx=to_dev(in_idx), out_idx=to_dev(act))
            bond = np.where(span > 0, hi_c + 1, lo_c).astype(np.int32)
            r_idx = u_c * E + bond if use_env else np.zeros(cnt)
            # left environment: L_lo (no support), else the last ping-pong buffer
            for grp, base, l_idx in (
                    (span == 0, Lflat, u_c * E + lo_c if use_env else np.zeros(cnt)),
                    ((span > 0) & (span % 2 == 1), cur[0], np.arange(cnt)),
                    ((span > 0) & (span % 2 == 0), cur[1], np.arange(cnt))):
                sel = np.nonzero(grp)[0]
                if len(sel) == 0:
                    continue
                part = torch.empty(len(sel), dtype=torch.complex128, device=dev)
                # keep every index tensor referenced until the launch is queued (a freed
                # temporary's block could be refilled by the next copy before the kernel runs)
                d_s, d_b = to_dev(state_idx[c0:c1][sel]), to_dev(bond[sel])
                d_l, d_r = to_dev(l_idx[sel]), to_dev(r_idx[sel])
                rc = self.lib.bmps_env_close(
                    _ptr(self.dims), n, cap, d_s.data_ptr(), d_b.data_ptr(), base.data_ptr(), cc,
                    d_l.data_ptr(), Rflat.data_ptr(), cc, d_r.data_ptr(), len(sel), part.data_ptr(),
                    _stream())
                _native.check(rc, "bmps_env_close")
                out[c0 + sel] = part.cpu().numpy()
        bad = np.abs(out.imag) > 1e-10
        if bad.any():
            raise RuntimeError(f"expectation has imaginary residue {out.imag[bad][0]:.3e}")
        return out.real.copy()

    # -- stats --------------------------------------------------------------------
    def stats(self) -> dict:
        self.check_status()
        return {
            "trunc_error_sq": self.trunc_err.cpu().numpy(),
            "peak_entries": self.peak.cpu().numpy(),
            "max_bond_seen": self.mbs.cpu().numpy(),
            "entries": self.entries.cpu().numpy(),
            "min_margin": self.min_margin.cpu().numpy(),
            "min_gap": self.min_gap.cpu().numpy(),
        }
