"""Column-sharded bi-level projection across ranks (one process per GPU).

For a matrix too large for one GPU -- or already sharded by columns, like a
tensor-parallel weight -- each rank holds a contiguous column block
Y[:, c0:c1] as its own row-major (n, m_local) array.  The projection
(proj/src/bilevel.cpp:10-32) then has exactly one exchange step
(SURVEY.md §8e):

    1. local column q-norms v_local           (K1, no communication)
    2. all-gather of the m-length norm vector  (torch.distributed; NCCL over
                                               NVLink on GPUs, ~8 B/column)
    3. outer p-ball projection of v, redundantly on every rank (deterministic,
       so every rank derives identical budgets)
    4. local apply at budgets u[c0:c1]          (K3 / K3b, no communication)

Every per-column quantity is computed from the same column and the outer
projection sees the same vector, so the result equals the single-device
projection of the whole matrix: bit for bit for l_inf column maxima (exact),
to f64 rounding of the column sums for l1 / l2 (their row grouping follows
the grid, which depends on the block width).

``ShardedBilevelProjector`` plans once (the only host sync: one all-gather of
the block widths) and then projects with no host synchronisation, no
allocation in the C-ABI calls and exactly one collective per call
(``all_gather_into_tensor`` of the fixed-width padded norm blocks), so a call
can sit inside a captured CUDA graph next to the training step.

The local compute is a pluggable backend: ``CudaBackend`` drives the sm_100a
kernels through the C-ABI (the product path).  Tests may pass a CPU backend
built on the oracle to exercise the sharding logic with gloo on CPU.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _capi


class CudaBackend:
    """Local steps on torch CUDA tensors through the C-ABI (mp_aggregate,
    mp_project_ball, mp_project_fibers).  ``plan`` sizes every workspace once;
    the per-call methods write into caller-provided outputs and never sync."""

    def __init__(self, device=None):
        import torch
        self.torch = torch
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.lib = _capi.lib()
        self.ws = None

    def plan(self, n: int, m_local: int, m: int, dt: int, p: int, q: int):
        t, L = self.torch, self.lib
        need = max(L.mp_aggregate_workspace_size(dt, n, m_local, q),
                   L.mp_project_ball_workspace_size(_capi.MP_F64, m, p),
                   L.mp_project_fibers_workspace_size(dt, n, m_local, q), 256)
        self.ws = t.empty(int(need), dtype=t.uint8, device=self.device)
        self.info = t.zeros(C.sizeof(_capi.MpInfo), dtype=t.uint8, device=self.device)

    def _stream(self):
        self.torch.cuda.set_device(self.device)  # the C-ABI launches on the current device
        return self.torch.cuda.current_stream(self.device).cuda_stream

    def norms(self, y_local, q: int, out):
        n, m = y_local.shape
        _capi.check(self.lib.mp_aggregate(y_local.data_ptr(), out.data_ptr(), _dtype_code(y_local), n, m, q,
                                          self.ws.data_ptr(), self.ws.numel(), self._stream()))
        return out

    def outer(self, v, p: int, eta: float, out):
        _capi.check(self.lib.mp_project_ball(v.data_ptr(), out.data_ptr(), _capi.MP_F64, v.numel(), p, float(eta),
                                             self.info.data_ptr(), self.ws.data_ptr(), self.ws.numel(),
                                             self._stream()))
        return out

    def apply(self, y_local, x_local, q: int, v_local, u_local, flags: int = 0):
        n, m = y_local.shape
        _capi.check(self.lib.mp_project_fibers(y_local.data_ptr(), x_local.data_ptr(), _dtype_code(y_local), n, m,
                                               q, v_local.data_ptr(), u_local.data_ptr(), flags,
                                               self.ws.data_ptr(), self.ws.numel(), self._stream()))
        return x_local

    def status(self) -> int:
        """Device status of the last outer projection (syncs)."""
        return _capi.MpInfo.from_buffer_copy(self.info.cpu().numpy().tobytes()).status


def _dtype_code(t) -> int:
    import torch
    if t.dtype == torch.float32:
        return _capi.MP_F32
    if t.dtype == torch.float64:
        return _capi.MP_F64
    raise _capi.MpConfigError(f"unsupported dtype {t.dtype}")


class ShardedBilevelProjector:
    """Planned column-sharded bi-level projection; every rank of ``group``
    constructs one and calls it collectively.

    ``__call__(y_local, x_local, eta)`` writes this rank's projected block
    into x_local (may be y_local).  Per call: local K1, one
    ``all_gather_into_tensor`` of the norm blocks padded to the widest block,
    the outer projection on every rank, the local apply, and an on-device
    zero-column count -- no host sync, nothing allocated by the C-ABI."""

    def __init__(self, n: int, m_local: int, dtype, p="1", q="inf", group=None, backend=None, flags: int = 0,
                 device=None):
        import torch
        import torch.distributed as td
        self.group, self.flags = group, flags
        self.pc, self.qc = _capi.norm_code(p), _capi.norm_code(q)
        self.n, self.m_local = int(n), int(m_local)
        self.world, self.rank = td.get_world_size(group), td.get_rank(group)
        self.be = backend or CudaBackend(device)
        dev = getattr(self.be, "device", torch.device("cpu"))
        # plan-time exchange of block widths (the only host sync)
        mine = torch.tensor([self.m_local], dtype=torch.int64, device=dev)
        widths = torch.empty(self.world, dtype=torch.int64, device=dev)
        td.all_gather_into_tensor(widths, mine, group=group)
        self.widths = [int(w) for w in widths.cpu().tolist()]
        self.c0 = sum(self.widths[:self.rank])
        self.m = sum(self.widths)
        self.pad = max(self.widths)
        f64 = dict(dtype=torch.float64, device=dev)
        self.send = torch.zeros(self.pad, **f64)
        self.recv = torch.empty(self.world * self.pad, **f64)
        if all(w == self.pad for w in self.widths):
            self.index = None
            self.v = self.recv
        else:
            idx = [r * self.pad + k for r, w in enumerate(self.widths) for k in range(w)]
            self.index = torch.tensor(idx, dtype=torch.int64, device=dev)
            self.v = torch.empty(self.m, **f64)
        self.u = torch.empty(self.m, **f64)
        self.zero_count = torch.zeros((), dtype=torch.int64, device=dev)
        dt = _dtype_code(torch.empty(0, dtype=dtype))
        if hasattr(self.be, "plan"):
            self.be.plan(self.n, self.m_local, self.m, dt, self.pc, self.qc)

    def __call__(self, y_local, x_local, eta: float):
        import torch
        import torch.distributed as td
        if not (eta >= 0.0) or not np.isfinite(eta):
            raise _capi.MpValueError("radius must be a finite nonnegative real")
        if tuple(y_local.shape) != (self.n, self.m_local):
            raise _capi.MpShapeError(f"planned for a ({self.n}, {self.m_local}) block, got {tuple(y_local.shape)}")
        v_local = self.send[:self.m_local]
        self.be.norms(y_local, self.qc, v_local)
        td.all_gather_into_tensor(self.recv, self.send, group=self.group)
        if self.index is not None:
            torch.index_select(self.recv, 0, self.index, out=self.v)
        self.be.outer(self.v, self.pc, eta, self.u)
        self.be.apply(y_local, x_local, self.qc, v_local, self.budgets, self.flags)
        torch.sum((self.u == 0) | (self.v == 0), dim=0, out=self.zero_count)
        return x_local

    @property
    def budgets(self):
        """This rank's slice of the budgets u (device tensor, no copy)."""
        return self.u[self.c0:self.c0 + self.m_local]

    def zero_columns(self) -> int:
        """Global zeroed-column count of the last call (syncs; raises the
        outer projection's device status if it failed)."""
        if hasattr(self.be, "status"):
            _capi.check(self.be.status())
        return int(self.zero_count.item())


def sharded_bilevel_project(y_local, eta: float, p="1", q="inf", backend=None, group=None, flags: int = 0):
    """One-shot form: plan, project, and read the zero count.

    Returns (x_local, budgets_local, zero_columns_global).  Every rank must
    call it (collective); blocks are concatenated in rank order."""
    if not (eta >= 0.0) or not np.isfinite(eta):
        raise _capi.MpValueError("radius must be a finite nonnegative real")
    n, m_local = y_local.shape
    proj = ShardedBilevelProjector(n, m_local, y_local.dtype, p, q, group=group, backend=backend, flags=flags,
                                   device=getattr(y_local, "device", None))
    x_local = proj(y_local, y_local.clone(), eta)
    return x_local, proj.budgets.clone(), proj.zero_columns()
