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
    mp_project_ball, mp_project_fibers)."""

    def __init__(self, device=None):
        import torch
        self.torch = torch
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.lib = _capi.lib()

    def _ws(self, nbytes):
        return self.torch.empty(max(int(nbytes), 256), dtype=self.torch.uint8, device=self.device)

    def norms(self, y_local, q: int):
        t = self.torch
        n, m = y_local.shape
        dt = _capi.MP_F32 if y_local.dtype == t.float32 else _capi.MP_F64
        out = t.empty(m, dtype=t.float64, device=self.device)
        ws = self._ws(self.lib.mp_aggregate_workspace_size(dt, n, m, q))
        s = t.cuda.current_stream(self.device)
        _capi.check(self.lib.mp_aggregate(y_local.data_ptr(), out.data_ptr(), dt, n, m, q, ws.data_ptr(), ws.numel(),
                                          s.cuda_stream))
        return out

    def outer(self, v, p: int, eta: float):
        t = self.torch
        u = t.empty_like(v)
        ws = self._ws(self.lib.mp_project_ball_workspace_size(_capi.MP_F64, v.numel(), p))
        info = t.zeros(C.sizeof(_capi.MpInfo), dtype=t.uint8, device=self.device)
        s = t.cuda.current_stream(self.device)
        _capi.check(self.lib.mp_project_ball(v.data_ptr(), u.data_ptr(), _capi.MP_F64, v.numel(), p, float(eta),
                                             info.data_ptr(), ws.data_ptr(), ws.numel(), s.cuda_stream))
        st = _capi.MpInfo.from_buffer_copy(info.cpu().numpy().tobytes()).status
        _capi.check(st)
        return u

    def apply(self, y_local, x_local, q: int, v_local, u_local, flags: int = 0):
        t = self.torch
        n, m = y_local.shape
        dt = _capi.MP_F32 if y_local.dtype == t.float32 else _capi.MP_F64
        ws = self._ws(self.lib.mp_project_fibers_workspace_size(dt, n, m, q))
        s = t.cuda.current_stream(self.device)
        _capi.check(self.lib.mp_project_fibers(y_local.data_ptr(), x_local.data_ptr(), dt, n, m, q,
                                               v_local.contiguous().data_ptr(), u_local.contiguous().data_ptr(),
                                               flags, ws.data_ptr(), ws.numel(), s.cuda_stream))
        return x_local

    def gather(self, v_local, group=None):
        return gather_norms(v_local, group)


def gather_norms(v_local, group=None):
    """All-gather variable-length norm vectors (torch tensors) in rank order."""
    import torch
    import torch.distributed as td
    world = td.get_world_size(group)
    dev = v_local.device
    sizes = torch.tensor([v_local.numel()], dtype=torch.int64, device=dev)
    all_sizes = [torch.zeros_like(sizes) for _ in range(world)]
    td.all_gather(all_sizes, sizes, group=group)
    mx = int(max(int(s.item()) for s in all_sizes))
    pad = torch.zeros(mx, dtype=v_local.dtype, device=dev)
    pad[:v_local.numel()] = v_local
    parts = [torch.empty_like(pad) for _ in range(world)]
    td.all_gather(parts, pad, group=group)
    return torch.cat([parts[r][:int(all_sizes[r].item())] for r in range(world)])


def sharded_bilevel_project(y_local, eta: float, p="1", q="inf", backend=None, group=None, flags: int = 0):
    """Project the global matrix whose column block this rank holds.

    Returns (x_local, budgets_local, zero_columns_global).  Every rank must
    call it (collective); blocks are concatenated in rank order."""
    import torch.distributed as td
    pc, qc = _capi.norm_code(p), _capi.norm_code(q)
    if not (eta >= 0.0) or not np.isfinite(eta):
        raise _capi.MpValueError("radius must be a finite nonnegative real")
    be = backend or CudaBackend(getattr(y_local, "device", None))
    rank = td.get_rank(group)
    v_local = be.norms(y_local, qc)
    v = be.gather(v_local, group)
    # offsets of this rank's block in the gathered vector
    import torch
    world = td.get_world_size(group)
    counts = torch.tensor([v_local.numel()], dtype=torch.int64, device=v_local.device)
    all_counts = [torch.zeros_like(counts) for _ in range(world)]
    td.all_gather(all_counts, counts, group=group)
    c0 = int(sum(int(c.item()) for c in all_counts[:rank]))
    u = be.outer(v, pc, eta)
    u_local = u[c0:c0 + v_local.numel()]
    x_local = be.apply(y_local, y_local.clone(), qc, v_local, u_local, flags)
    zero_columns = int(((u == 0) | (v == 0)).sum().item())
    return x_local, u_local, zero_columns
