"""ctypes binding of ``libbmps.so`` (the C ABI declared in ``include/bmps.h``).

The library is built in-tree by ``paper_1807_07914_b200/build.py`` (or
``__graft_entry__.build()``). There is no CPU fallback: importing a compute
entry point without the library, or without a CUDA device, raises.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "libbmps.so"

BMPS_S_OK = 0
BMPS_S_SVD_FAILED = 1
BMPS_S_ALL_TRUNCATED = 2
BMPS_S_CAPACITY = 3
BMPS_PLAN_E_SITE = -10
BMPS_PLAN_E_SAME_SITE = -11


class BmpsPolicy(ctypes.Structure):
    _fields_ = [("cutoff", ctypes.c_double), ("max_bond", ctypes.c_int32), ("relative", ctypes.c_int32)]


class BmpsParams(ctypes.Structure):
    """``bmps_params`` (include/bmps.h): every tunable of one bmps_apply_2q call."""

    _fields_ = [("tol_factor", ctypes.c_double), ("max_sweeps", ctypes.c_int32),
                ("max_inner", ctypes.c_int32), ("qr_min_cols", ctypes.c_int32),
                ("jacobi_mode", ctypes.c_int32), ("block_w2", ctypes.c_int32),
                ("double_qr", ctypes.c_int32), ("col_sort", ctypes.c_int32),
                ("gram_cache", ctypes.c_int32), ("pair_skip", ctypes.c_int32),
                ("jac_cluster", ctypes.c_int32), ("jac_per_sm", ctypes.c_int32),
                ("jac_ws", ctypes.c_int32), ("tma_staging", ctypes.c_int32),
                ("cluster_size", ctypes.c_int32), ("qr_cluster", ctypes.c_int32),
                ("n_svd_events", ctypes.c_int32),
                ("svd_events", ctypes.c_void_p), ("svd_events_used", ctypes.c_void_p),
                ("thr_a", ctypes.c_double), ("thr_b", ctypes.c_double),
                ("thr_a_sweeps", ctypes.c_int32), ("thr_b_sweeps", ctypes.c_int32),
                ("thr_auto", ctypes.c_int32), ("qr_small", ctypes.c_int32),
                ("visits_hint", ctypes.c_int32)]


RECORD_BYTES = 48  # sizeof(bmps_update_record)

_P = ctypes.c_void_p
_I = ctypes.c_int32
_SZ = ctypes.c_size_t
_L = ctypes.c_int64

_SIGNATURES = {
    "bmps_version": ([], _I),
    "bmps_status_string": ([_I], ctypes.c_char_p),
    "bmps_launch_count": ([], ctypes.c_uint64),
    "bmps_build_flags": ([], _I),
    "bmps_default_params": ([_P], None),
    "bmps_phase_cycles": ([_P], _I),
    "bmps_inner_trace": ([_P, _I], _I),
    "bmps_debug_inner_sweep": ([_P, _P, _P, _I, ctypes.c_double, ctypes.c_double, ctypes.c_double, _I, _P, _P], _I),
    "bmps_init_product": ([_P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _I, _I, _P], _I),
    "bmps_apply_1q": ([_P, _P, _I, _I, _I, _P, _P, _I, _P], _I),
    "bmps_apply_2q_workspace_bytes": ([_I, _I], _SZ),
    "bmps_apply_2q": ([_P, _P, _P, _I, _I, _I, _P, _P, _I, BmpsPolicy, _P, _P, _P, _SZ, _I, _P, _P], _I),
    "bmps_stats_replay": ([_P, _P, _I, _P, _P, _P, _P, _P, _P, _P, _I, _P, _P, _P], _I),
    "bmps_conditional": ([_P, _P, _P, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P], _I),
    "bmps_apply_2q_sweeps": ([_P, _I, _P, _P], _I),
    "bmps_amplitudes": ([_P, _P, _P, _I, _I, _I, _P, _P, _I, _P, _P], _I),
    "bmps_sample": ([_P, _P, _P, _I, _I, _I, _P, _P, _I, _P, _P], _I),
    "bmps_env_transfer": ([_P, _P, _P, _I, _I, _I, _P, _P, _P, _I, _P, _L, _P, _P, _L, _P, _P, _I, _P], _I),
    "bmps_env_close": ([_P, _I, _I, _P, _P, _P, _L, _P, _P, _L, _P, _I, _P, _P], _I),
    "bmps_env_sweep": ([_P, _P, _P, _I, _I, _I, _P, _I, _I, _P, _L, _P], _I),
    "bmps_pauli_sweep": ([_P, _P, _P, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _L, _I, _P, _P], _I),
    "bmps_plan_expanded_count": ([_P, _P, _P, _L], _L),
    "bmps_plan_build": ([_I, _P, _P, _P, _P, _P, _I, _P, _P, _P, _P, _P, _P, _P], _I),
    "bmps_dense_init": ([_P, _I, _I, _P], _I),
    "bmps_dense_apply_1q": ([_P, _I, _I, _P, _P], _I),
    "bmps_dense_apply_2q": ([_P, _I, _I, _I, _P, _P], _I),
    "bmps_dense_run_smem": ([_P, _I, _I, _P, _P, _I, _P], _I),
    "bmps_dense_expect_workspace_bytes": ([_I], _SZ),
    "bmps_dense_expect": ([_P, _I, _I, _P, _P, _P, _I, _P, _SZ, _P, _P], _I),
    "bmps_dense_prob_tree": ([_P, _I, _P, _P], _I),
    "bmps_dense_sample": ([_P, _I, _P, _I, _P, _P], _I),
}

EXPORTED = tuple(_SIGNATURES)

_lib = None


# tunables of bmps_apply_2q (bmps_default_params); the package-level overrides
# below apply to every call made while they are set (the library itself keeps no
# mutable state: each call gets its own bmps_params)
TUNABLES = ("tol_factor", "max_sweeps", "max_inner", "qr_min_cols", "jacobi_mode", "block_w2",
            "double_qr", "col_sort", "gram_cache", "pair_skip", "jac_cluster", "jac_per_sm",
            "jac_ws", "tma_staging", "cluster_size", "qr_cluster", "thr_a", "thr_b", "thr_a_sweeps",
            "thr_b_sweeps", "thr_auto", "qr_small", "visits_hint")
_overrides: dict = {}


def experimental() -> bool:
    """True when libbmps.so was built with -DBMPS_EXPERIMENTAL (slower development variants)."""
    return bool(load().bmps_build_flags() & 1)


_param_cache: dict = {}


def params(**extra) -> BmpsParams:
    """A ``bmps_params`` of the library defaults, the active overrides and ``extra``
    (a fresh struct; the default-plus-overrides part is memoised per override set)."""
    key = tuple(sorted({**_overrides, **extra}.items()))
    base = _param_cache.get(key)
    if base is not None:
        p = BmpsParams()
        ctypes.pointer(p)[0] = base
        return p
    p = BmpsParams()
    load().bmps_default_params(ctypes.byref(p))
    for k, v in {**_overrides, **extra}.items():
        if k not in TUNABLES:
            raise ValueError(f"unknown tunable {k!r}")
        setattr(p, k, type(getattr(p, k))(v))
    saved = BmpsParams()
    ctypes.pointer(saved)[0] = p
    _param_cache[key] = saved
    return p


def default_params() -> dict:
    p = BmpsParams()
    load().bmps_default_params(ctypes.byref(p))
    return {k: getattr(p, k) for k in TUNABLES}


class tunables:
    """``with tunables(jac_cluster=4): ...`` -- override Jacobi tunables for the calls
    made inside the block (tests, A/B tools)."""

    def __init__(self, **kw):
        for k in kw:
            if k not in TUNABLES:
                raise ValueError(f"unknown tunable {k!r}")
        self.kw = kw
        self.saved: dict = {}

    def __enter__(self):
        self.saved = dict(_overrides)
        _overrides.update(self.kw)
        return self

    def __exit__(self, *exc):
        _overrides.clear()
        _overrides.update(self.saved)
        return False


_DEV_AIDS = ("bmps_phase_cycles", "bmps_inner_trace", "bmps_debug_inner_sweep")   # timer-build diagnostics, not the product ABI


def load(path: str | os.PathLike | None = None) -> ctypes.CDLL:
    """Load libbmps.so and declare every exported signature (no device needed)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    # BMPS_LIB: an alternative build of the same ABI (A/B runs of development variants)
    p = Path(path) if path is not None else Path(os.environ.get("BMPS_LIB") or LIB_PATH)
    if not p.exists():
        raise RuntimeError(
            f"libbmps.so not found at {p}; build it with `python -m paper_1807_07914_b200.build` "
            "(there is no CPU fallback)"
        )
    lib = ctypes.CDLL(str(p))
    for name, (args, res) in _SIGNATURES.items():
        if name in _DEV_AIDS and os.environ.get("BMPS_LIB") and not hasattr(lib, name):
            continue   # an older development variant under A/B (BMPS_LIB) may lack a dev aid
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    if path is None:
        _lib = lib
        # optional tunables, e.g. BMPS_PARAMS="block_w2=64,tol_factor=4"
        for kv in filter(None, os.environ.get("BMPS_PARAMS", "").split(",")):
            k, v = kv.split("=")
            k = k.strip()
            if k not in TUNABLES:
                raise ValueError(f"bad BMPS_PARAMS entry {kv!r}")
            _overrides[k] = float(v)
    return lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load().bmps_status_string(rc).decode()
        raise RuntimeError(f"{what} failed: {msg} (code {rc})")
