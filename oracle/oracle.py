"""ctypes front for the CPU checker (TEST INFRASTRUCTURE ONLY).

Two backends, both f64 and CPU-only:

* ``liboracle.so`` -- our plain-C restatement (``oracle/mp_oracle.c``) of the
  reference algorithms, each function citing the reference file:line it
  follows.
* ``_ref/libmultiproj_ref.so`` -- the unmodified reference library compiled
  from /root/reference/proj/src by ``oracle/Makefile`` (present when it was
  built; it travels to the GPU box as a prebuilt file).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this module, and only as the checker or
the CPU baseline.  The product package never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import sys
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
NORMS = {"1": 0, "2": 1, "inf": 2}

_P_D = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_P_F = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_P_I64 = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_P_I32 = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_P_U64 = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")


class OracleError(ValueError):
    """Mirrors the reference ValueError/ShapeError/ConfigError family."""

    def __init__(self, code: int):
        self.code = code
        super().__init__({1: "ValueError", 2: "ShapeError", 3: "ConfigError"}.get(code, f"error {code}"))


def _check(rc: int) -> None:
    if rc != 0:
        raise OracleError(rc)


def build(ref: bool | None = None) -> None:
    """Compile liboracle.so (and _ref when the reference sources exist)."""
    targets = ["all"]
    if ref is None:
        ref = os.path.isdir("/root/reference/proj/src")
    if ref:
        targets += ["ref", "suites"]
    subprocess.run(["make", "-s", "-j8", "-C", HERE, f"PYTHON={sys.executable}"] + targets, check=True)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            build(ref=False)
        L = C.CDLL(path)
        L.orc_aggregate.argtypes = [_P_D, C.c_int64, C.c_int64, C.c_int, _P_D]
        L.orc_aggregate.restype = None
        L.orc_project_l1_inplace.argtypes = [_P_D, C.c_int64, C.c_double, C.POINTER(C.c_double), C.POINTER(C.c_int64)]
        L.orc_project_l1_inplace.restype = None
        L.orc_project_l1_sort_inplace.argtypes = L.orc_project_l1_inplace.argtypes
        L.orc_project_l1_sort_inplace.restype = None
        L.orc_project_ball.argtypes = [_P_D, C.c_int64, C.c_int, C.c_double]
        L.orc_project_ball.restype = C.c_int
        L.orc_bilevel.argtypes = [_P_D, C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_double,
                                  _P_D, _P_D, _P_D, C.POINTER(C.c_int64), C.POINTER(C.c_double)]
        L.orc_bilevel.restype = C.c_int
        L.orc_multilevel.argtypes = [_P_D, _P_I64, C.c_int, _P_I32, C.c_double, _P_D, C.c_void_p]
        L.orc_multilevel.restype = C.c_int
        L.orc_multilevel_norm.argtypes = [_P_D, _P_I64, C.c_int, _P_I32, C.POINTER(C.c_double)]
        L.orc_multilevel_norm.restype = C.c_int
        L.orc_vector_norm.argtypes = [_P_D, C.c_int64, C.c_int, C.POINTER(C.c_double)]
        L.orc_vector_norm.restype = C.c_int
        L.orc_project_fibers.argtypes = [_P_D, C.c_int64, C.c_int64, C.c_int, _P_D, _P_D]
        L.orc_project_fibers.restype = None
        L.orc_structured_sparsity.argtypes = [_P_D, C.c_int64, C.c_int64, C.c_double]
        L.orc_structured_sparsity.restype = C.c_int64
        L.orc_euclid_l1inf.argtypes = [_P_D, C.c_int64, C.c_int64, C.c_double, _P_D, _P_D, C.POINTER(C.c_double)]
        L.orc_euclid_l1inf.restype = C.c_int
        L.orc_clip_cost.argtypes = [_P_D, C.c_int64, C.c_int64, _P_D]
        L.orc_clip_cost.restype = C.c_double
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(os.path.join(HERE, "_ref", "libmultiproj_ref.so"))


def ref():
    """The compiled reference (oracle/_ref).  Raises if it was never built."""
    global _ref
    if _ref is None:
        path = os.path.join(HERE, "_ref", "libmultiproj_ref.so")
        R = C.CDLL(path)
        R.ref_bilevel.argtypes = [_P_D, C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_double, C.c_int,
                                  _P_D, _P_D, C.POINTER(C.c_int64)]
        R.ref_bilevel.restype = C.c_int
        R.ref_time_bilevel.argtypes = [_P_F, C.c_int64, C.c_int64, C.c_int, C.c_int, _P_D, C.c_int,
                                       C.c_int, C.c_int, _P_D]
        R.ref_time_bilevel.restype = C.c_int
        R.ref_multilevel.argtypes = [_P_D, _P_I64, C.c_int, _P_I32, C.c_int, C.c_double, C.c_int,
                                     _P_D, C.c_void_p]
        R.ref_multilevel.restype = C.c_int
        R.ref_multilevel_recursive.argtypes = [_P_D, _P_I64, C.c_int, _P_I32, C.c_int, C.c_double, _P_D]
        R.ref_multilevel_recursive.restype = C.c_int
        R.ref_trilevel_l1infinf.argtypes = [_P_D, _P_I64, C.c_double, _P_D]
        R.ref_trilevel_l1infinf.restype = C.c_int
        R.ref_project_ball.argtypes = [_P_D, C.c_int64, C.c_int, C.c_double, C.c_int, _P_D]
        R.ref_project_ball.restype = C.c_int
        R.ref_multilevel_norm.argtypes = [_P_D, _P_I64, C.c_int, _P_I32, C.c_int, C.POINTER(C.c_double)]
        R.ref_multilevel_norm.restype = C.c_int
        R.ref_gen_uniform.argtypes = [C.c_uint64, C.c_double, C.c_double, _P_D, C.c_int64]
        R.ref_gen_uniform.restype = None
        R.ref_gen_normal.argtypes = [C.c_uint64, _P_D, C.c_int64]
        R.ref_gen_normal.restype = None
        R.ref_gen_raw.argtypes = [C.c_uint64, _P_U64, C.c_int64]
        R.ref_gen_raw.restype = None
        R.ref_euclid.argtypes = [_P_D, C.c_int64, C.c_int64, C.c_double, _P_D, _P_D, C.POINTER(C.c_double)]
        R.ref_euclid.restype = C.c_int
        R.ref_budget_grid.argtypes = [_P_D, C.c_int64, C.c_int64, C.c_double, C.c_int64, _P_D,
                                      C.POINTER(C.c_double)]
        R.ref_budget_grid.restype = C.c_int
        R.ref_clip_cost.argtypes = [_P_D, C.c_int64, C.c_int64, _P_D]
        R.ref_clip_cost.restype = C.c_double
        R.ref_write_uniform_tensor.argtypes = [C.c_char_p, _P_I64, C.c_int, C.c_uint64, C.c_double, C.c_double,
                                               C.POINTER(C.c_uint64)]
        R.ref_write_uniform_tensor.restype = C.c_int
        R.ref_read_tensor_checksum.argtypes = [C.c_char_p, C.POINTER(C.c_uint64), C.POINTER(C.c_int64)]
        R.ref_read_tensor_checksum.restype = C.c_int
        R.ref_rng_stream.argtypes = [C.c_uint64, C.c_int, _P_U64, _P_D]
        R.ref_rng_stream.restype = C.c_int
        R.ref_write_records_sample.argtypes = [C.c_char_p]
        R.ref_write_records_sample.restype = C.c_int
        _ref = R
    return _ref


def _d(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _norm(q) -> int:
    return NORMS[q] if isinstance(q, str) else int(q)


# ----------------------------------------------------------------- restatement
def aggregate(t, q) -> np.ndarray:
    t = _d(t)
    n = t.shape[0]
    m = t.size // n
    out = np.empty(m, np.float64)
    lib().orc_aggregate(t.reshape(-1), n, m, _norm(q), out)
    return out.reshape(t.shape[1:])


def project_l1(y, radius, sort: bool = False):
    """Returns (x, tau, k); tau = k = -1 when y was already feasible."""
    x = _d(y).copy().reshape(-1)
    tau, k = C.c_double(), C.c_int64()
    fn = lib().orc_project_l1_sort_inplace if sort else lib().orc_project_l1_inplace
    fn(x, x.size, float(radius), C.byref(tau), C.byref(k))
    return x, tau.value, k.value


def project_ball(y, q, radius) -> np.ndarray:
    x = _d(y).copy()
    _check(lib().orc_project_ball(x.reshape(-1), x.size, _norm(q), float(radius)))
    return x


def bilevel(y, eta, p="1", q="inf"):
    """Returns dict(X, budgets, v, zero_columns, tau)."""
    y = _d(y)
    if y.ndim != 2:
        raise OracleError(2)
    n, m = y.shape
    x = np.empty_like(y)
    b = np.empty(m, np.float64)
    v = np.empty(m, np.float64)
    z, tau = C.c_int64(), C.c_double(-1.0)
    _check(lib().orc_bilevel(y.reshape(-1), n, m, _norm(p), _norm(q), float(eta), x.reshape(-1), b, v,
                             C.byref(z), C.byref(tau)))
    return {"X": x, "budgets": b, "v": v, "zero_columns": z.value, "tau": tau.value}


def _chain_sizes(shape):
    sizes = []
    for i in range(len(shape) - 1, 0, -1):
        sizes.append(int(np.prod(shape[i:])))
    return sizes


def multilevel(t, levels, eta, want_chain: bool = False):
    t = _d(t)
    lv = np.asarray([_norm(q) for q in levels], np.int32)
    if len(lv) != t.ndim:
        raise OracleError(2)
    shape = np.asarray(t.shape, np.int64)
    x = np.empty_like(t)
    sizes = _chain_sizes(t.shape)
    chain = np.empty(max(1, sum(sizes)), np.float64) if want_chain else None
    _check(lib().orc_multilevel(t.reshape(-1), shape, t.ndim, lv, float(eta), x.reshape(-1),
                                chain.ctypes.data if chain is not None else None))
    if not want_chain:
        return x
    out, off = [], 0
    for i, s in zip(range(t.ndim - 1, 0, -1), sizes):
        out.append(chain[off:off + s].reshape(t.shape[i:]))
        off += s
    return x, out


def multilevel_norm(t, levels) -> float:
    t = _d(t)
    lv = np.asarray([_norm(q) for q in levels], np.int32)
    out = C.c_double()
    _check(lib().orc_multilevel_norm(t.reshape(-1), np.asarray(t.shape, np.int64), t.ndim, lv, C.byref(out)))
    return out.value


def matrix_pq_norm(y, p, q) -> float:
    return multilevel_norm(y, [q, p])


def project_fibers(y, q, v, budgets):
    """Columns of y projected onto q-balls of radii budgets given norms v."""
    x = _d(y).copy()
    lib().orc_project_fibers(x.reshape(-1), x.shape[0], x.size // x.shape[0], _norm(q), _d(v), _d(budgets))
    return x


def structured_sparsity(x, tol=0.0) -> int:
    x = _d(x)
    return int(lib().orc_structured_sparsity(x.reshape(-1), x.shape[0], x.size // x.shape[0], float(tol)))


# --------------------------------------------------------- compiled reference
def euclid(y, eta):
    """Exact Euclidean l1,inf projection (proj/src/euclidean.cpp:82-170):
    returns (X, budgets, theta)."""
    y = _d(y)
    n, m = y.shape
    x = np.empty_like(y)
    b = np.empty(m)
    th = C.c_double()
    _check(lib().orc_euclid_l1inf(y, n, m, float(eta), x, b, C.byref(th)))
    return x, b, th.value


def clip_cost(y, budgets) -> float:
    y = _d(y)
    return float(lib().orc_clip_cost(y, y.shape[0], y.shape[1], _d(budgets)))


def ref_euclid(y, eta):
    y = _d(y)
    n, m = y.shape
    x = np.empty_like(y)
    b = np.empty(m)
    th = C.c_double()
    _check(ref().ref_euclid(y, n, m, float(eta), x, b, C.byref(th)))
    return x, b, th.value


def ref_budget_grid(y, eta, steps):
    y = _d(y)
    n, m = y.shape
    b = np.empty(m)
    th = C.c_double()
    _check(ref().ref_budget_grid(y, n, m, float(eta), int(steps), b, C.byref(th)))
    return b, th.value


def ref_clip_cost(y, budgets) -> float:
    y = _d(y)
    return float(ref().ref_clip_cost(y, y.shape[0], y.shape[1], _d(budgets)))


def ref_write_uniform_tensor(path, shape, seed, lo=-1.0, hi=1.0) -> int:
    sh = np.ascontiguousarray(shape, np.int64)
    ck = C.c_uint64()
    _check(ref().ref_write_uniform_tensor(str(path).encode(), sh, len(shape), seed, lo, hi, C.byref(ck)))
    return ck.value


def ref_read_tensor_checksum(path):
    ck, sz = C.c_uint64(), C.c_int64()
    _check(ref().ref_read_tensor_checksum(str(path).encode(), C.byref(ck), C.byref(sz)))
    return ck.value, sz.value


def ref_rng_stream(seed, count):
    raw = np.empty(count, np.uint64)
    nrm = np.empty(count)
    _check(ref().ref_rng_stream(seed, count, raw, nrm))
    return raw, nrm


def ref_write_records_sample(path) -> None:
    _check(ref().ref_write_records_sample(str(path).encode()))


def ref_bilevel(y, eta, p="1", q="inf", workers=1):
    y = _d(y)
    n, m = y.shape
    x = np.empty_like(y)
    b = np.empty(m, np.float64)
    z = C.c_int64()
    _check(ref().ref_bilevel(y.reshape(-1), n, m, _norm(p), _norm(q), float(eta), int(workers), x.reshape(-1), b,
                             C.byref(z)))
    return {"X": x, "budgets": b, "zero_columns": z.value}


def ref_multilevel(t, levels, eta, workers=1, want_chain=False, recursive=False):
    t = _d(t)
    lv = np.asarray([_norm(q) for q in levels], np.int32)
    shape = np.asarray(t.shape, np.int64)
    x = np.empty_like(t)
    if recursive:
        _check(ref().ref_multilevel_recursive(t.reshape(-1), shape, t.ndim, lv, len(lv), float(eta), x.reshape(-1)))
        return x
    sizes = _chain_sizes(t.shape)
    chain = np.empty(max(1, sum(sizes)), np.float64) if want_chain else None
    _check(ref().ref_multilevel(t.reshape(-1), shape, t.ndim, lv, len(lv), float(eta), int(workers), x.reshape(-1),
                                chain.ctypes.data if chain is not None else None))
    if not want_chain:
        return x
    out, off = [], 0
    for i, s in zip(range(t.ndim - 1, 0, -1), sizes):
        out.append(chain[off:off + s].reshape(t.shape[i:]))
        off += s
    return x, out


def ref_trilevel(t, eta):
    t = _d(t)
    x = np.empty_like(t)
    _check(ref().ref_trilevel_l1infinf(t.reshape(-1), np.asarray(t.shape, np.int64), float(eta), x.reshape(-1)))
    return x


def ref_project_ball(y, q, radius, sort=False):
    y = _d(y).reshape(-1)
    out = np.empty_like(y)
    _check(ref().ref_project_ball(y, y.size, _norm(q), float(radius), int(sort), out))
    return out


def ref_multilevel_norm(t, levels):
    t = _d(t)
    lv = np.asarray([_norm(q) for q in levels], np.int32)
    out = C.c_double()
    _check(ref().ref_multilevel_norm(t.reshape(-1), np.asarray(t.shape, np.int64), t.ndim, lv, len(lv),
                                     C.byref(out)))
    return out.value


def ref_gen_uniform(seed, count, lo=0.0, hi=1.0):
    out = np.empty(count, np.float64)
    ref().ref_gen_uniform(seed, lo, hi, out, count)
    return out


def ref_gen_normal(seed, count):
    out = np.empty(count, np.float64)
    ref().ref_gen_normal(seed, out, count)
    return out


def ref_gen_raw(seed, count):
    out = np.empty(count, np.uint64)
    ref().ref_gen_raw(seed, out, count)
    return out


def ref_time_bilevel(y32, etas, p="1", q="inf", reps=1, workers=1):
    """Seconds per reference bilevel_project call (bench_one recipe)."""
    y32 = np.ascontiguousarray(y32, np.float32)
    n, m = y32.shape
    etas = np.asarray(etas, np.float64)
    times = np.empty(len(etas) * reps, np.float64)
    _check(ref().ref_time_bilevel(y32.reshape(-1), n, m, _norm(p), _norm(q), etas, len(etas), reps, workers, times))
    return times
