"""Seeded synthetic inputs for the five BASELINE.json configs (harness only).

Thin ctypes front of ``libmp_datagen.so`` (csrc/datagen.c), which restates
the reference generator (SplitMix64 -> xoshiro256++, proj/src/rng.cpp) so the
GPU path and the CPU reference consume byte-identical fp32 inputs.  Seeds
follow SURVEY.md §8d: configs 1-5 use seeds 1-5.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _build

_lib = None
KIND_UNIFORM, KIND_NORMAL, KIND_LAPLACE = 0, 1, 2


def _L():
    global _lib
    if _lib is None:
        if not os.path.exists(_build.DATAGEN):
            _build.build()
        L = C.CDLL(_build.DATAGEN)
        L.mpg_generate.argtypes = [C.c_uint64, C.c_int, C.c_double, C.c_double, C.c_int64, C.c_void_p, C.c_void_p]
        L.mpg_generate.restype = None
        L.mpg_raw.argtypes = [C.c_uint64, C.c_void_p, C.c_int64]
        L.mpg_raw.restype = None
        _lib = L
    return _lib


def _gen(seed, kind, a, b, shape, dtype):
    count = int(np.prod(shape))
    out = np.empty(count, dtype=dtype)
    p32 = out.ctypes.data if out.dtype == np.float32 else None
    p64 = out.ctypes.data if out.dtype == np.float64 else None
    _L().mpg_generate(int(seed), kind, float(a), float(b), count, p32, p64)
    return out.reshape(shape)


def uniform(seed, shape, lo=0.0, hi=1.0, dtype=np.float32):
    return _gen(seed, KIND_UNIFORM, lo, hi, shape, dtype)


def normal(seed, shape, dtype=np.float32):
    return _gen(seed, KIND_NORMAL, 0.0, 0.0, shape, dtype)


def laplace(seed, shape, b, dtype=np.float32):
    return _gen(seed, KIND_LAPLACE, b, 0.0, shape, dtype)


def raw(seed, count):
    out = np.empty(count, np.uint64)
    _L().mpg_raw(int(seed), out.ctypes.data, count)
    return out


# ------------------------------------------------------------ the configs
def config_input(cfg: int, scale: float = 1.0):
    """fp32 input of BASELINE.json config `cfg` (1-5).  `scale` < 1 shrinks
    the leading dims for quick tests (same distribution and seed)."""
    def dim(d):
        return max(2, int(round(d * scale)))
    if cfg == 1:
        return normal(1, (dim(1000), dim(1000)))
    if cfg == 2:
        return uniform(2, (dim(10000), dim(10000)), -1.0, 1.0)
    if cfg == 3:
        return normal(3, (dim(4096), dim(16384)))
    if cfg == 4:
        return normal(4, (dim(256), dim(256), dim(256)))
    if cfg == 5:
        return laplace(5, (dim(32768), dim(8192)), 0.01)
    raise ValueError(cfg)


def config5_eta(colmax: np.ndarray, frac: float = 0.9) -> float:
    """eta zeroing ~frac of the columns at iteration 0: v sorted
    ascending (0-based), k = floor(frac*m), t* = (v[k] + v[k+1])/2 -- the
    midpoint, so no column sits at tau -- and eta = sum_j max(v_j - t*, 0).
    Columns v[0..k] (k+1 of them; 7373 of 8192) are zeroed at iteration 0."""
    v = np.sort(np.asarray(colmax, np.float64))
    k = int(np.floor(frac * v.size))
    t = 0.5 * (v[k] + v[k + 1])
    return float(np.sum(np.maximum(v - t, 0.0)))
