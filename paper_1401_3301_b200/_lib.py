"""ctypes binding of include/simplex_asm_b200.h.

Loading never falls back to anything: if the sm_100a library is missing the
import of the device layer raises ExtensionMissingError.
"""

from __future__ import annotations

import ctypes
import os

from . import _build
from .errors import (
    CapacityError,
    DegenerateSimplexError,
    ExtensionMissingError,
    IndexRangeError,
)

SA_OK, SA_ERR_DEGENERATE, SA_ERR_INDEX_RANGE, SA_ERR_CAPACITY, SA_ERR_ARG, SA_ERR_CUDA, SA_ERR_NOMEM = range(7)
SA_OP_MASS, SA_OP_STIFF, SA_OP_ELASTIC, SA_OP_GENERAL = 1, 2, 4, 8
SA_OP_EXACT = 16
SA_CORE = {"SkylakeX": 0, "Haswell": 1}

# every symbol include/simplex_asm_b200.h declares
EXPORTS = (
    "sa_mesh_create", "sa_mesh_create_split", "sa_host_narrow_upload", "sa_host_widen_i32", "sa_mesh_vols", "sa_mesh_validate",
    "sa_mesh_destroy",
    "sa_plan_create", "sa_plan_info", "sa_plan_stats", "sa_plan_pattern", "sa_plan_destroy",
    "sa_numeric", "sa_compact", "sa_unpack_columns", "sa_plan_prepare", "sa_mesh_set_coords", "sa_kuhn_mesh", "sa_kuhn_slab",
    "sa_pk_plan_create", "sa_pk_plan_info", "sa_pk_plan_pattern", "sa_pk_mass", "sa_pk_compact", "sa_pk_plan_destroy",
    "sa_last_error", "sa_bad_index", "sa_launch_count",
)


class SaCoeffs(ctypes.Structure):
    _fields_ = [
        ("w", ctypes.c_void_p), ("w_const", ctypes.c_double),
        ("lamb", ctypes.c_void_p), ("lamb_const", ctypes.c_double),
        ("mu", ctypes.c_void_p), ("mu_const", ctypes.c_double),
        ("A", ctypes.c_void_p), ("b", ctypes.c_void_p), ("c", ctypes.c_void_p), ("a0", ctypes.c_void_p),
        ("A_const", ctypes.c_double * 9), ("a0_const", ctypes.c_double),
        ("gen_packed", ctypes.c_void_p),
        ("lambs_e", ctypes.c_void_p),
        ("mus_e", ctypes.c_void_p),
    ]


_lib = None


def lib_path() -> str:
    return _build.LIB_PATH


def load(build_if_missing: bool = True):
    """Load (building first if stale and nvcc is present) the library."""
    global _lib
    if _lib is not None:
        return _lib
    path = _build.LIB_PATH
    override = os.environ.get("SA_LIB_PATH")   # A/B experiments: a prebuilt variant
    if override:
        path, build_if_missing = override, False
    if build_if_missing:
        try:
            _build.build()
        except Exception as exc:  # no nvcc on this machine
            if not os.path.exists(path):
                raise ExtensionMissingError(f"cannot build {path}: {exc}") from exc
    if not os.path.exists(path):
        raise ExtensionMissingError(f"sm_100a library {path} is missing; run __graft_entry__.build()")
    L = ctypes.CDLL(path)
    vp, i64, i64p, dp = ctypes.c_void_p, ctypes.c_int64, ctypes.POINTER(ctypes.c_int64), ctypes.c_void_p
    L.sa_mesh_create.argtypes = [ctypes.c_int, i64, i64, vp, vp, vp, ctypes.c_int, ctypes.c_int, vp,
                                 ctypes.POINTER(vp)]
    L.sa_mesh_create_split.argtypes = [ctypes.c_int, i64, i64, vp, vp, ctypes.c_int, vp, vp, ctypes.c_int, ctypes.c_int,
                                       vp, ctypes.POINTER(vp)]
    L.sa_host_narrow_upload.argtypes = [vp, i64, i64, vp, vp, ctypes.c_int, ctypes.c_int, vp, i64p]
    L.sa_host_widen_i32.argtypes = [vp, i64, i64, vp, ctypes.c_int]
    L.sa_mesh_vols.argtypes = [vp, vp, vp]
    L.sa_mesh_validate.argtypes = [vp, vp, i64p, i64p, vp]
    L.sa_mesh_destroy.argtypes = [vp]
    L.sa_plan_create.argtypes = [vp, ctypes.c_int, i64, i64, vp, ctypes.POINTER(vp)]
    L.sa_plan_info.argtypes = [vp, i64p, i64p, i64p]
    L.sa_plan_stats.argtypes = [vp, i64p, ctypes.c_int]
    L.sa_plan_pattern.argtypes = [vp, vp, vp, vp]
    L.sa_plan_destroy.argtypes = [vp]
    L.sa_numeric.argtypes = [vp, ctypes.c_int, ctypes.POINTER(SaCoeffs), ctypes.POINTER(vp), i64p, vp]
    L.sa_plan_prepare.argtypes = [vp, ctypes.c_int, vp]
    L.sa_unpack_columns.argtypes = [vp, ctypes.c_int, vp, vp, i64, vp, vp]
    L.sa_mesh_set_coords.argtypes = [vp, vp, vp, vp]
    L.sa_pk_plan_create.argtypes = [ctypes.c_int, i64, i64, vp, ctypes.c_int, vp, ctypes.POINTER(vp)]
    L.sa_pk_plan_info.argtypes = [vp, i64p, i64p]
    L.sa_pk_plan_pattern.argtypes = [vp, vp, vp, vp]
    L.sa_pk_mass.argtypes = [vp, vp, vp, vp, i64p, vp]
    L.sa_pk_compact.argtypes = [vp, vp, vp, vp, vp, vp]
    L.sa_pk_plan_destroy.argtypes = [vp]
    u64 = ctypes.c_uint64
    L.sa_kuhn_mesh.argtypes = [ctypes.c_int, i64, ctypes.c_int, ctypes.c_double, ctypes.c_double, u64, u64, u64, u64,
                               vp, vp, vp]
    L.sa_kuhn_slab.argtypes = [ctypes.c_int, i64, ctypes.c_int, ctypes.c_double, ctypes.c_double, u64, u64, u64, u64,
                               i64, i64, i64, i64, vp, vp, vp]
    L.sa_compact.argtypes = [vp, vp, vp, vp, vp, vp]
    L.sa_last_error.restype = ctypes.c_char_p
    L.sa_bad_index.restype = ctypes.c_int64
    L.sa_launch_count.restype = ctypes.c_int64
    L.sa_launch_count.argtypes = [ctypes.c_int]
    for name in EXPORTS:
        getattr(L, name).restype = getattr(L, name).restype if name in (
            "sa_last_error", "sa_bad_index", "sa_launch_count") else ctypes.c_int
    _lib = L
    return L


def check(rc: int) -> None:
    """Map an sa_status to the reference's exception types (errors.py)."""
    if rc == SA_OK:
        return
    L = load(build_if_missing=False)
    msg = (L.sa_last_error() or b"").decode(errors="replace")
    if rc == SA_ERR_DEGENERATE:
        raise DegenerateSimplexError(int(L.sa_bad_index()))
    if rc == SA_ERR_INDEX_RANGE:
        raise IndexRangeError(msg)
    if rc == SA_ERR_CAPACITY:
        raise CapacityError(msg)
    if rc == SA_ERR_ARG:
        raise ValueError(msg)
    if rc == SA_ERR_NOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"simplex_asm_b200: {msg} (status {rc})")
