"""ctypes binding of the C-ABI in include/mp_cuda.h (libmp_b200.so).

The library is REQUIRED: there is no CPU fallback.  If it is missing the
import raises, and every call fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

from . import _build

MP_OK, MP_ERR_VALUE, MP_ERR_SHAPE, MP_ERR_CONFIG, MP_ERR_CUDA, MP_ERR_WORKSPACE, MP_ERR_UNSUPPORTED = range(7)
MP_NORM = {"1": 0, "2": 1, "inf": 2}
MP_F32, MP_F64 = 0, 1
MP_FLAG_EXACT_ZERO_SIGN = 1

# Every exported symbol of include/mp_cuda.h (checked by tests/test_capi.py).
EXPORTS = [
    "mp_bilevel_workspace_size", "mp_bilevel_project",
    "mp_multilevel_workspace_size", "mp_multilevel_project",
    "mp_project_ball_workspace_size", "mp_project_ball",
    "mp_aggregate_workspace_size", "mp_aggregate",
    "mp_project_fibers_workspace_size", "mp_project_fibers",
    "mp_euclid_workspace_size", "mp_euclid_project", "mp_euclid_project_host",
    "mp_context_create", "mp_context_destroy",
    "mp_bilevel_project_host", "mp_bilevel_sweep_host", "mp_bilevel_sweep_host_async", "mp_context_wait",
    "mp_multilevel_project_host",
    "mp_project_ball_host", "mp_aggregate_host", "mp_perturb_gaussian",
    "mp_profile_events", "mp_profile_timeline", "mp_last_error", "mp_version",
]


class MpInfo(C.Structure):
    _fields_ = [("tau", C.c_double), ("zero_columns", C.c_int64), ("active", C.c_int64),
                ("survivors", C.c_int64), ("status", C.c_int32), ("iterations", C.c_int32)]


class ProjectionError(ValueError):
    """Base of the mirrored reference exceptions (pybind maps them all to
    Python ValueError, proj/python/bindings.cpp:46-48)."""


class MpValueError(ProjectionError):
    pass


class MpShapeError(ProjectionError):
    pass


class MpConfigError(ProjectionError):
    pass


class MpCudaError(RuntimeError):
    pass


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_build.LIB):
        raise ImportError(f"{_build.LIB} is missing: run paper_2405_02086_b200._build.build() "
                          "(there is no CPU fallback)")
    L = C.CDLL(_build.LIB)
    i64, vp, dbl, u32 = C.c_int64, C.c_void_p, C.c_double, C.c_uint
    sz, st, en = C.c_size_t, C.c_int, C.c_int
    L.mp_bilevel_workspace_size.argtypes = [en, i64, i64, en, en]
    L.mp_bilevel_workspace_size.restype = sz
    L.mp_bilevel_project.argtypes = [vp, vp, en, i64, i64, en, en, dbl, vp, vp, vp, u32, vp, sz, vp]
    L.mp_bilevel_project.restype = st
    L.mp_multilevel_workspace_size.argtypes = [en, vp, C.c_int, vp, C.c_int]
    L.mp_multilevel_workspace_size.restype = sz
    L.mp_multilevel_project.argtypes = [vp, vp, en, vp, C.c_int, vp, C.c_int, dbl, vp, vp, u32, vp, sz, vp]
    L.mp_multilevel_project.restype = st
    L.mp_project_ball_workspace_size.argtypes = [en, i64, en]
    L.mp_project_ball_workspace_size.restype = sz
    L.mp_project_ball.argtypes = [vp, vp, en, i64, en, dbl, vp, vp, sz, vp]
    L.mp_project_ball.restype = st
    L.mp_aggregate_workspace_size.argtypes = [en, i64, i64, en]
    L.mp_aggregate_workspace_size.restype = sz
    L.mp_aggregate.argtypes = [vp, vp, en, i64, i64, en, vp, sz, vp]
    L.mp_aggregate.restype = st
    L.mp_project_fibers_workspace_size.argtypes = [en, i64, i64, en]
    L.mp_project_fibers_workspace_size.restype = sz
    L.mp_project_fibers.argtypes = [vp, vp, en, i64, i64, en, vp, vp, u32, vp, sz, vp]
    L.mp_project_fibers.restype = st
    L.mp_euclid_workspace_size.argtypes = [en, i64, i64]
    L.mp_euclid_workspace_size.restype = sz
    L.mp_euclid_project.argtypes = [vp, vp, en, i64, i64, dbl, vp, vp, u32, vp, sz, vp]
    L.mp_euclid_project.restype = st
    L.mp_euclid_project_host.argtypes = [vp, vp, vp, en, i64, i64, dbl, vp, vp]
    L.mp_euclid_project_host.restype = st
    L.mp_context_create.argtypes = [C.c_int]
    L.mp_context_create.restype = vp
    L.mp_context_destroy.argtypes = [vp]
    L.mp_context_destroy.restype = None
    L.mp_bilevel_project_host.argtypes = [vp, vp, vp, en, i64, i64, en, en, dbl, vp, vp, vp, u32]
    L.mp_bilevel_project_host.restype = st
    L.mp_bilevel_sweep_host.argtypes = [vp, vp, vp, en, i64, i64, en, en, vp, C.c_int, vp, vp, u32]
    L.mp_bilevel_sweep_host.restype = st
    L.mp_bilevel_sweep_host_async.argtypes = [vp, vp, vp, en, i64, i64, en, en, vp, C.c_int, vp, vp, u32, vp]
    L.mp_bilevel_sweep_host_async.restype = st
    L.mp_context_wait.argtypes = [vp, C.c_uint64]
    L.mp_context_wait.restype = st
    L.mp_multilevel_project_host.argtypes = [vp, vp, vp, en, vp, C.c_int, vp, C.c_int, dbl, vp, u32]
    L.mp_multilevel_project_host.restype = st
    L.mp_project_ball_host.argtypes = [vp, vp, vp, en, i64, en, dbl]
    L.mp_project_ball_host.restype = st
    L.mp_aggregate_host.argtypes = [vp, vp, vp, en, i64, i64, en]
    L.mp_aggregate_host.restype = st
    L.mp_profile_events.argtypes = [C.c_void_p, C.c_int]
    L.mp_profile_events.restype = None
    L.mp_perturb_gaussian.argtypes = [vp, en, i64, dbl, C.c_uint64, C.c_uint64, vp]
    L.mp_perturb_gaussian.restype = st
    L.mp_profile_timeline.argtypes = [C.c_void_p]
    L.mp_profile_timeline.restype = None
    L.mp_last_error.argtypes = []
    L.mp_last_error.restype = C.c_char_p
    L.mp_version.argtypes = []
    L.mp_version.restype = C.c_int
    _lib = L
    return L


def check(status: int) -> None:
    if status == MP_OK:
        return
    msg = (lib().mp_last_error() or b"").decode(errors="replace")
    if status == MP_ERR_VALUE:
        raise MpValueError(msg)
    if status == MP_ERR_SHAPE:
        raise MpShapeError(msg)
    if status == MP_ERR_CONFIG:
        raise MpConfigError(msg)
    if status == MP_ERR_CUDA:
        raise MpCudaError(msg)
    raise RuntimeError(f"mp status {status}: {msg}")


def norm_code(q) -> int:
    if isinstance(q, int):
        return q
    try:
        return MP_NORM[str(q)]
    except KeyError:
        raise MpConfigError(f"bad norm token '{q}' (expected 1, 2 or inf)") from None


def parse_norm_spec(spec: str) -> list[int]:
    """'inf,inf,1' -> codes, innermost first (proj/src/multilevel.cpp:20-41)."""
    if isinstance(spec, (list, tuple)):
        return [norm_code(q) for q in spec]
    return [norm_code(tok) for tok in spec.split(",")]
