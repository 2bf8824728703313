"""B200-native bi-level / multi-level norm-ball projections (arXiv 2405.02086).

Python host mirror of the reference module ``multiproj``
(proj/python/bindings.cpp:51-137, proj/python/multiproj/__init__.py): same
function names, argument meaning and error behaviour, computed by the sm_100a
kernels of ``libmp_b200.so`` through the C-ABI (include/mp_cuda.h).

* numpy inputs take the host path (``mp_*_host``: host->device copy, kernels,
  device->host copy).  float32 arrays stay float32 (the fp32 device path);
  anything else is force-cast to float64 like the reference binding
  (proj/python/bindings.cpp:17-25).
* torch CUDA tensors take the device path (no copies, current torch stream).

There is no CPU fallback: without the CUDA library every call raises.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _capi
from ._capi import (MP_F32, MP_F64, MP_FLAG_EXACT_ZERO_SIGN, MpInfo, MpConfigError, MpShapeError, MpValueError,
                    ProjectionError, check, lib, norm_code, parse_norm_spec)

__all__ = [
    "bilevel_project", "bilevel_radius_sweep", "multilevel_project", "trilevel_project_l1infinf", "project_l1", "project_l2",
    "project_linf", "project_ball", "euclid_project_l1inf", "matrix_pq_norm", "multilevel_norm", "aggregate_leading_axis",
    "structured_sparsity", "gen_uniform_matrix", "perturb_gaussian", "BilevelProjector", "MultilevelProjector",
    "ProjectionError", "MpValueError", "MpShapeError", "MpConfigError", "MP_FLAG_EXACT_ZERO_SIGN",
]


def _is_torch(a) -> bool:
    return type(a).__module__.startswith("torch")


def _is_cuda_tensor(a) -> bool:
    """torch CUDA tensors take the device path; CPU tensors are host arrays."""
    return _is_torch(a) and a.device.type == "cuda"


def _host_array(a) -> np.ndarray:
    arr = a.detach().numpy() if _is_torch(a) else np.asarray(a)
    if arr.dtype != np.float32:
        arr = arr.astype(np.float64)
    return np.ascontiguousarray(arr)


def _dt(arr) -> int:
    if _is_torch(arr):
        import torch
        if arr.dtype == torch.float32:
            return MP_F32
        if arr.dtype == torch.float64:
            return MP_F64
        raise MpConfigError(f"unsupported dtype {arr.dtype}")
    return MP_F32 if arr.dtype == np.float32 else MP_F64


def _torch_dtype(dtype):
    """Strict dtype map for the device projectors: float32 / float64 only.

    Anything else (float16, bfloat16, integers) would have the kernels read
    and write 8-byte elements through a 2- or 4-byte buffer, so it raises."""
    import torch
    if dtype in (torch.float32, "float32", "torch.float32", np.float32):
        return torch.float32, MP_F32
    if dtype in (torch.float64, "float64", "torch.float64", np.float64):
        return torch.float64, MP_F64
    raise MpConfigError(f"unsupported dtype {dtype}: the projections compute in float32 or float64")


def _check_operand(t, name, shape, tdtype, device):
    import torch
    if not isinstance(t, torch.Tensor) or t.device.type != "cuda":
        raise MpConfigError(f"{name} must be a CUDA tensor")
    if t.device != device:
        raise MpConfigError(f"{name} is on {t.device}, the projector was planned for {device}")
    if t.dtype != tdtype:
        raise MpConfigError(f"{name} has dtype {t.dtype}, the projector was planned for {tdtype}")
    if tuple(t.shape) != tuple(shape):
        raise MpShapeError(f"{name} has shape {tuple(t.shape)}, the projector was planned for {tuple(shape)}")
    if not t.is_contiguous():
        raise MpConfigError(f"{name} must be contiguous (row-major fibers)")


def _ptr(a) -> int:
    return a.data_ptr() if _is_torch(a) else a.ctypes.data


# -------------------------------------------------------------- device path
def _cuda_device(device):
    import torch
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    d = torch.device(device)
    if d.type != "cuda":
        raise MpConfigError(f"device projectors run on CUDA devices, not {d}")
    return torch.device("cuda", d.index if d.index is not None else torch.cuda.current_device())


class BilevelProjector:
    """Pre-planned bi-level projection on device tensors.

    Owns its workspace so a call allocates nothing and never syncs: it can be
    captured in a CUDA graph.  ``__call__(y, x, eta)`` writes x (may be y)."""

    def __init__(self, n: int, m: int, dtype="float32", p="1", q="inf", device=None, flags: int = 0):
        import torch
        self.n, self.m = int(n), int(m)
        self.tdtype, self.dt = _torch_dtype(dtype)
        self.p, self.q = norm_code(p), norm_code(q)
        self.flags = flags
        self.device = _cuda_device(device)
        wsb = lib().mp_bilevel_workspace_size(self.dt, self.n, self.m, self.p, self.q)
        if wsb == 0:
            raise MpShapeError("bilevel_project requires a non-empty order-2 tensor")
        self.ws = torch.empty(wsb, dtype=torch.uint8, device=self.device)
        self.budgets = torch.empty(self.m, dtype=torch.float64, device=self.device)
        self.norms = torch.empty(self.m, dtype=torch.float64, device=self.device)
        self.info_buf = torch.zeros(C.sizeof(MpInfo), dtype=torch.uint8, device=self.device)

    def __call__(self, y, x, eta: float, stream=None):
        import torch
        _check_operand(y, "y", (self.n, self.m), self.tdtype, self.device)
        _check_operand(x, "x", (self.n, self.m), self.tdtype, self.device)
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        with torch.cuda.device(self.device):  # the C-ABI launches on the current device
            check(lib().mp_bilevel_project(y.data_ptr(), x.data_ptr(), self.dt, self.n, self.m, self.p, self.q,
                                           float(eta), self.budgets.data_ptr(), self.norms.data_ptr(),
                                           self.info_buf.data_ptr(), self.flags, self.ws.data_ptr(),
                                           self.ws.numel(), s.cuda_stream))
        return x

    def info(self) -> MpInfo:
        raw = self.info_buf.cpu().numpy().tobytes()
        return MpInfo.from_buffer_copy(raw)


class MultilevelProjector:
    """Pre-planned multi-level projection on device tensors (graph capturable)."""

    def __init__(self, shape, levels, dtype="float32", device=None, flags: int = 0, want_chain: bool = True):
        import torch
        self.want_chain = want_chain  # False lets (inf, ..., inf, p) specs collapse to one bi-level pass
        self.shape = [int(s) for s in shape]
        self.levels = parse_norm_spec(levels)
        self.tdtype, self.dt = _torch_dtype(dtype)
        self.flags = flags
        self.device = _cuda_device(device)
        self._shape_c = (C.c_int64 * len(self.shape))(*self.shape)
        self._lv_c = (C.c_int * max(1, len(self.levels)))(*self.levels)
        wsb = lib().mp_multilevel_workspace_size(self.dt, self._shape_c, len(self.shape), self._lv_c,
                                                 len(self.levels))
        if wsb == 0:
            # reproduce the reference's error for this spec / shape
            check(lib().mp_multilevel_project(None, None, self.dt, self._shape_c, len(self.shape), self._lv_c,
                                              len(self.levels), 0.0, None, None, 0, None, 0, None))
        self.ws = torch.empty(wsb, dtype=torch.uint8, device=self.device)
        chain = 0
        for i in range(len(self.shape) - 1, 0, -1):
            chain += int(np.prod(self.shape[i:]))
        self.chain = torch.empty(max(1, chain), dtype=torch.float64, device=self.device)
        self.info_buf = torch.zeros(C.sizeof(MpInfo), dtype=torch.uint8, device=self.device)

    def __call__(self, t, x, eta: float, stream=None):
        import torch
        _check_operand(t, "t", self.shape, self.tdtype, self.device)
        _check_operand(x, "x", self.shape, self.tdtype, self.device)
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        with torch.cuda.device(self.device):
            check(lib().mp_multilevel_project(t.data_ptr(), x.data_ptr(), self.dt, self._shape_c, len(self.shape),
                                              self._lv_c, len(self.levels), float(eta),
                                              self.chain.data_ptr() if self.want_chain else None,
                                              self.info_buf.data_ptr(), self.flags, self.ws.data_ptr(),
                                              self.ws.numel(), s.cuda_stream))
        return x

    def budget_chain(self):
        out, off = [], 0
        for i in range(len(self.shape) - 1, 0, -1):
            size = int(np.prod(self.shape[i:]))
            out.append(self.chain[off:off + size].reshape(self.shape[i:]))
            off += size
        return out

    def info(self) -> MpInfo:
        return MpInfo.from_buffer_copy(self.info_buf.cpu().numpy().tobytes())


# ------------------------------------------------------------ public API
def bilevel_project(y, eta, p="1", q="inf", workers=1, flags: int = 0):
    """Bi-level l_{p,q} projection; returns (X, budgets, zero_columns).

    Mirrors ``multiproj.bilevel_project`` (proj/python/bindings.cpp:71-85 ->
    proj/src/bilevel.cpp:10-32).  ``workers`` is accepted for API
    compatibility; the CUDA grid replaces the CPU pool."""
    del workers
    pc, qc = norm_code(p), norm_code(q)
    if _is_cuda_tensor(y):
        if y.dim() != 2:
            raise MpShapeError("bilevel_project requires order 2")
        yc = y.contiguous()
        proj = BilevelProjector(yc.shape[0], yc.shape[1], yc.dtype, pc, qc, yc.device, flags)
        x = proj(yc, yc.clone(), eta)
        info = proj.info()
        check(info.status)
        return x, proj.budgets.clone(), int(info.zero_columns)
    arr = _host_array(y)
    if arr.ndim != 2:
        raise MpShapeError("bilevel_project requires order 2")
    n, m = arr.shape
    x = np.empty_like(arr)
    budgets = np.empty(m, np.float64)
    z, tau = C.c_int64(), C.c_double()
    check(lib().mp_bilevel_project_host(None, arr.ctypes.data, x.ctypes.data, _dt(arr), n, m, pc, qc, float(eta),
                                        budgets.ctypes.data, C.addressof(z), C.addressof(tau), flags))
    return x, budgets.tolist(), int(z.value)


def bilevel_radius_sweep(y, etas, p="1", q="inf", flags: int = 0):
    """Project one host matrix at several radii (the reference's radius sweep,
    proj/src/bench.cpp:93-106): one upload, downloads overlapped with the next
    projection.  Returns a list of (X, budgets, zero_columns)."""
    pc, qc = norm_code(p), norm_code(q)
    arr = _host_array(y)
    if arr.ndim != 2:
        raise MpShapeError("bilevel_project requires order 2")
    n, m = arr.shape
    etas = np.ascontiguousarray(etas, np.float64)
    xs = [np.empty_like(arr) for _ in etas]
    ptrs = (C.c_void_p * len(xs))(*[x.ctypes.data for x in xs])
    budgets = np.empty((len(etas), m), np.float64)
    zeros = np.empty(len(etas), np.int64)
    check(lib().mp_bilevel_sweep_host(None, arr.ctypes.data, ptrs, _dt(arr), n, m, pc, qc, etas.ctypes.data,
                                      len(etas), budgets.ctypes.data, zeros.ctypes.data, flags))
    return [(xs[k], budgets[k].tolist(), int(zeros[k])) for k in range(len(etas))]


def multilevel_project(y, norms, eta, workers=1, flags: int = 0, return_chain: bool = False):
    """Multi-level projection, norms innermost first (e.g. 'inf,inf,1').

    Mirrors ``multiproj.multilevel_project`` (proj/python/bindings.cpp:87-99
    -> multilevel_project_iter, proj/src/multilevel.cpp:93-124)."""
    del workers
    levels = parse_norm_spec(norms)
    if _is_cuda_tensor(y):
        t = y.contiguous()
        proj = MultilevelProjector(t.shape, levels, t.dtype, t.device, flags)
        x = proj(t, t.clone(), eta)
        check(proj.info().status)
        return (x, proj.budget_chain()) if return_chain else x
    arr = _host_array(y)
    if arr.ndim == 0:
        raise MpShapeError("tensor order must be >= 1")
    shape = (C.c_int64 * arr.ndim)(*arr.shape)
    lv = (C.c_int * max(1, len(levels)))(*levels)
    x = np.empty_like(arr)
    sizes = [int(np.prod(arr.shape[i:])) for i in range(arr.ndim - 1, 0, -1)]
    chain = np.empty(max(1, sum(sizes)), np.float64)
    check(lib().mp_multilevel_project_host(None, arr.ctypes.data, x.ctypes.data, _dt(arr), shape, arr.ndim, lv,
                                           len(levels), float(eta), chain.ctypes.data if return_chain else None,
                                           flags))
    if not return_chain:
        return x
    out, off = [], 0
    for i, s in zip(range(arr.ndim - 1, 0, -1), sizes):
        out.append(chain[off:off + s].reshape(arr.shape[i:]))
        off += s
    return x, out


def trilevel_project_l1infinf(t, eta, workers=1, flags: int = 0):
    """Named l_{1,inf,inf} path for order-3 tensors (proj/src/multilevel.cpp:126-132)."""
    nd = t.dim() if _is_torch(t) else np.asarray(t).ndim
    if nd != 3:
        raise MpShapeError("trilevel_project_l1infinf requires order 3")
    return multilevel_project(t, "inf,inf,1", eta, workers, flags)


def project_ball(y, q, radius):
    """Vector-ball projection (proj/src/vector_balls.cpp:207-214)."""
    qc = norm_code(q)
    arr = _host_array(y).reshape(-1)
    x = np.empty_like(arr)
    check(lib().mp_project_ball_host(None, arr.ctypes.data, x.ctypes.data, _dt(arr), arr.size, qc, float(radius)))
    return x


def project_l1(y, radius):
    return project_ball(y, "1", radius)


def project_l2(y, radius):
    return project_ball(y, "2", radius)


def project_linf(y, radius):
    return project_ball(y, "inf", radius)


def aggregate_leading_axis(t, q):
    """out[f] = ||fiber f||_q over the leading axis (proj/src/tensor.cpp:107-138)."""
    arr = _host_array(t)
    if arr.ndim < 2:
        raise MpShapeError("aggregate_leading_axis requires order >= 2")
    n = arr.shape[0]
    m = arr.size // n
    out = np.empty(m, np.float64)
    check(lib().mp_aggregate_host(None, arr.ctypes.data, out.ctypes.data, _dt(arr), n, m, norm_code(q)))
    return out.reshape(arr.shape[1:])


def _vector_norm(v: np.ndarray, q: int) -> float:
    # proj/src/tensor.cpp:78-99 on the (small) final aggregate
    if not np.all(np.isfinite(v)):
        raise MpValueError("non-finite vector entry")
    a = np.abs(v.astype(np.float64).reshape(-1))
    if q == 0:
        return float(np.sum(a))
    if q == 1:
        return float(np.sqrt(np.sum(a * a)))
    return float(np.max(a)) if a.size else 0.0


def multilevel_norm(y, norms) -> float:
    """Nested-norm value (proj/src/multilevel.cpp:134-141)."""
    levels = parse_norm_spec(norms)
    arr = _host_array(y)
    if len(levels) != arr.ndim:
        raise MpShapeError("norm spec depth does not match tensor order")
    if not np.all(np.isfinite(arr)):
        raise MpValueError("non-finite tensor entry")
    cur = arr
    for q in levels[:-1]:
        cur = aggregate_leading_axis(cur, q)
    return _vector_norm(cur, levels[-1])


def matrix_pq_norm(y, p, q) -> float:
    """||Y||_{p,q} (proj/src/tensor.cpp:101-105)."""
    arr = _host_array(y)
    if arr.ndim != 2:
        raise MpShapeError("matrix_pq_norm requires order 2")
    return multilevel_norm(arr, [norm_code(q), norm_code(p)])


def structured_sparsity(y, tol=0.0):
    """(zero_columns, fraction) of columns with max |x| <= tol (proj/src/tensor.cpp:152-164)."""
    arr = _host_array(y)
    if arr.ndim != 2:
        raise MpShapeError("structured_sparsity requires order 2")
    mx = aggregate_leading_axis(arr, "inf")
    count = int(np.sum(mx <= tol))
    return count, count / arr.shape[1]


def euclid_project_l1inf(y, eta):
    """Exact Euclidean l_{1,inf} projection; returns (X, budgets, theta).

    Mirrors ``multiproj.euclid_project_l1inf`` (proj/python/bindings.cpp:101-108
    -> proj/src/euclidean.cpp:82-170)."""
    if _is_cuda_tensor(y):
        import torch
        if y.dim() != 2:
            raise MpShapeError("euclid_project_l1inf requires order 2")
        yc = y.contiguous()
        n, m = yc.shape
        dt = _dt(yc)
        wsb = lib().mp_euclid_workspace_size(dt, n, m)
        ws = torch.empty(max(wsb, 256), dtype=torch.uint8, device=yc.device)
        x = torch.empty_like(yc)
        budgets = torch.empty(m, dtype=torch.float64, device=yc.device)
        info = torch.zeros(C.sizeof(MpInfo), dtype=torch.uint8, device=yc.device)
        s = torch.cuda.current_stream(yc.device)
        with torch.cuda.device(yc.device):
            check(lib().mp_euclid_project(yc.data_ptr(), x.data_ptr(), dt, n, m, float(eta), budgets.data_ptr(),
                                          info.data_ptr(), 0, ws.data_ptr(), wsb, s.cuda_stream))
        inf = MpInfo.from_buffer_copy(info.cpu().numpy().tobytes())
        check(inf.status)
        return x, budgets, float(inf.tau)
    arr = _host_array(y)
    if arr.ndim != 2:
        raise MpShapeError("euclid_project_l1inf requires order 2")
    n, m = arr.shape
    x = np.empty_like(arr)
    budgets = np.empty(m, np.float64)
    theta = C.c_double()
    check(lib().mp_euclid_project_host(None, arr.ctypes.data, x.ctypes.data, _dt(arr), n, m, float(eta),
                                       budgets.ctypes.data, C.addressof(theta)))
    return x, budgets.tolist(), float(theta.value)


def perturb_gaussian(x, sigma, seed, iteration, stream=None):
    """In-place x += sigma * N(0,1) on a torch CUDA tensor (config-5 loop
    harness; Philox4x32-10 keyed by (seed, iteration))."""
    import torch
    if not _is_cuda_tensor(x) or not x.is_contiguous():
        raise MpConfigError("perturb_gaussian needs a contiguous CUDA tensor")
    s = stream if stream is not None else torch.cuda.current_stream(x.device)
    with torch.cuda.device(x.device):
        check(lib().mp_perturb_gaussian(x.data_ptr(), _dt(x), x.numel(), float(sigma), int(seed), int(iteration),
                                        s.cuda_stream))
    return x


def gen_uniform_matrix(n, m, seed, lo=0.0, hi=1.0):
    """Deterministic uniform matrix (proj/src/rng.cpp:64-79), via datagen."""
    from . import datagen
    if n < 1 or m < 1:
        raise MpConfigError("matrix dims must be >= 1")
    if not lo < hi:
        raise MpConfigError("uniform bounds require lo < hi")
    return datagen.uniform(seed, (n, m), lo, hi, dtype=np.float64)
