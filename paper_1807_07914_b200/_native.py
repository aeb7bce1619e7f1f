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


RECORD_BYTES = 32  # sizeof(bmps_update_record)

_P = ctypes.c_void_p
_I = ctypes.c_int32
_SZ = ctypes.c_size_t
_L = ctypes.c_int64

_SIGNATURES = {
    "bmps_version": ([], _I),
    "bmps_status_string": ([_I], ctypes.c_char_p),
    "bmps_set_param": ([ctypes.c_char_p, ctypes.c_double], _I),
    "bmps_launch_count": ([], ctypes.c_uint64),
    "bmps_phase_cycles": ([_P], _I),
    "bmps_svd_time": ([_P, _P], _I),
    "bmps_debug_set_trace": ([_P], _I),
    "bmps_init_product": ([_P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _I, _I, _P], _I),
    "bmps_apply_1q": ([_P, _P, _I, _I, _I, _P, _P, _I, _P], _I),
    "bmps_apply_2q_workspace_bytes": ([_I, _I], _SZ),
    "bmps_apply_2q": ([_P, _P, _P, _I, _I, _I, _P, _P, _I, BmpsPolicy, _P, _P, _P, _SZ, _I, _I, _P], _I),
    "bmps_stats_replay": ([_P, _P, _I, _P, _P, _P, _P, _P, _P, _P], _I),
    "bmps_apply_2q_sweeps": ([_P, _I, _P, _P], _I),
    "bmps_amplitudes": ([_P, _P, _P, _I, _I, _I, _P, _P, _I, _P, _P], _I),
    "bmps_sample": ([_P, _P, _P, _I, _I, _I, _P, _P, _I, _P, _P], _I),
    "bmps_env_transfer": ([_P, _P, _P, _I, _I, _I, _P, _P, _P, _I, _P, _L, _P, _L, _P, _I, _P], _I),
    "bmps_env_close": ([_P, _I, _I, _P, _P, _P, _L, _P, _L, _I, _P, _P], _I),
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


# library defaults of the bmps_set_param tunables (csrc/bmps.cu)
DEFAULT_PARAMS = {"tol_factor": 4.0, "max_sweeps": 60, "max_inner": 1, "qr_min_cols": 65,
                  "jacobi_mode": 4, "cluster_size": 8, "tma_staging": 0, "gram_cache": 1,
                  "block_w2": 32, "double_qr": 1, "jac_per_sm": 0, "col_sort": 1, "time_svd": 0, "pair_skip": 1,
                  "jac_ws": 0, "jac_cluster": -1}


def load(path: str | os.PathLike | None = None) -> ctypes.CDLL:
    """Load libbmps.so and declare every exported signature (no device needed)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path is not None else LIB_PATH
    if not p.exists():
        raise RuntimeError(
            f"libbmps.so not found at {p}; build it with `python -m paper_1807_07914_b200.build` "
            "(there is no CPU fallback)"
        )
    lib = ctypes.CDLL(str(p))
    for name, (args, res) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    # optional tunables, e.g. BMPS_PARAMS="block_w2=64,tol_factor=4"
    for kv in filter(None, os.environ.get("BMPS_PARAMS", "").split(",")):
        k, v = kv.split("=")
        if lib.bmps_set_param(k.strip().encode(), float(v)) != 0:
            raise ValueError(f"bad BMPS_PARAMS entry {kv!r}")
    if path is None:
        _lib = lib
    return lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load().bmps_status_string(rc).decode()
        raise RuntimeError(f"{what} failed: {msg} (code {rc})")
