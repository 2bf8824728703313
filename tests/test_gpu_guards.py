"""Out-of-bounds write checks without compute-sanitizer: every device buffer
(input, output, workspace, budgets, info) is carved from one sentinel-filled
allocation with guard gaps, the kernels run at ragged shapes, and every guard
byte must still hold the sentinel afterwards; the input must be unchanged."""
import ctypes as C

import numpy as np
import pytest

import paper_2405_02086_b200 as mp
from paper_2405_02086_b200 import _capi

pytestmark = pytest.mark.gpu
GUARD = 4096
SENT = 0xA5


class Arena:
    def __init__(self, sizes):
        import torch
        self.torch = torch
        total = sum(((s + 255) // 256) * 256 + 2 * GUARD for s in sizes) + GUARD
        self.buf = torch.full((total,), SENT, dtype=torch.uint8, device="cuda")
        self.slices, off = [], GUARD
        for s in sizes:
            self.slices.append((off, s))
            off += ((s + 255) // 256) * 256 + 2 * GUARD
        self.ends = off

    def ptr(self, i):
        return self.buf.data_ptr() + self.slices[i][0]

    def view(self, i, dtype, shape):
        off, s = self.slices[i]
        return self.buf[off:off + s].view(dtype).view(shape)

    def check_guards(self):
        self.torch.cuda.synchronize()
        h = self.buf.cpu().numpy()
        prev = 0
        for off, s in self.slices:
            assert (h[prev:off] == SENT).all(), f"guard before slice at {off} overwritten"
            prev = off + s
        # tail of the last slice's rounding + guards up to the end
        assert (h[prev:] == SENT).all(), "trailing guard overwritten"


@pytest.mark.parametrize("dt", ["float32", "float64"])
# (600, 24) (1000, 8): 64-thread TMA strips; (1500, 16): 128-thread TMA strips;
# (3000, 8): 256-thread TMA strips (f32); (4097, 24): 512-thread TMA strips (f64)
@pytest.mark.parametrize("n,m", [(37, 45), (1, 7), (300, 64), (9000, 6), (4097, 24), (13000, 8), (5, 33),
                                 (600, 24), (1000, 8), (1500, 16), (3000, 8)])
def test_bilevel_writes_stay_in_bounds(dt, n, m):
    import torch
    lib = _capi.lib()
    tdt = getattr(torch, dt)
    code = _capi.MP_F32 if dt == "float32" else _capi.MP_F64
    s = 4 if dt == "float32" else 8
    rng = np.random.default_rng(n + m)
    y_h = rng.normal(size=(n, m)).astype(np.float32 if s == 4 else np.float64)
    for p in (0, 1, 2):
        for q in (0, 1, 2):
            wsb = lib.mp_bilevel_workspace_size(code, n, m, p, q)
            A = Arena([n * m * s, n * m * s, m * 8, m * 8, C.sizeof(_capi.MpInfo), wsb])
            y = A.view(0, tdt, (n, m))
            y.copy_(torch.from_numpy(y_h))
            eta = 0.3 * float(np.abs(y_h).max(axis=0).sum())
            _capi.check(lib.mp_bilevel_project(A.ptr(0), A.ptr(1), code, n, m, p, q, eta, A.ptr(2), A.ptr(3),
                                               A.ptr(4), 0, A.ptr(5), wsb, torch.cuda.current_stream().cuda_stream))
            A.check_guards()
            assert np.array_equal(y.cpu().numpy(), y_h)


def test_multilevel_euclid_fibers_in_bounds():
    import torch
    lib = _capi.lib()
    rng = np.random.default_rng(3)
    shape = (5, 6, 7)
    t_h = rng.normal(size=shape).astype(np.float32)
    for levels in ([2, 2, 0], [1, 0, 2], [0, 0, 0]):
        shp = (C.c_int64 * 3)(*shape)
        lv = (C.c_int * 3)(*levels)
        wsb = lib.mp_multilevel_workspace_size(_capi.MP_F32, shp, 3, lv, 3)
        chain = 6 * 7 + 7
        A = Arena([t_h.nbytes, t_h.nbytes, chain * 8, C.sizeof(_capi.MpInfo), wsb])
        A.view(0, torch.float32, shape).copy_(torch.from_numpy(t_h))
        _capi.check(lib.mp_multilevel_project(A.ptr(0), A.ptr(1), _capi.MP_F32, shp, 3, lv, 3, 0.5, A.ptr(2),
                                              A.ptr(3), 0, A.ptr(4), wsb, torch.cuda.current_stream().cuda_stream))
        A.check_guards()
    n, m = 77, 19
    y_h = rng.normal(size=(n, m)).astype(np.float32)
    wsb = lib.mp_euclid_workspace_size(_capi.MP_F32, n, m)
    A = Arena([y_h.nbytes, y_h.nbytes, m * 8, C.sizeof(_capi.MpInfo), wsb])
    A.view(0, torch.float32, (n, m)).copy_(torch.from_numpy(y_h))
    _capi.check(lib.mp_euclid_project(A.ptr(0), A.ptr(1), _capi.MP_F32, n, m, 2.0, A.ptr(2), A.ptr(3), 0, A.ptr(4),
                                      wsb, torch.cuda.current_stream().cuda_stream))
    A.check_guards()
    for q in (0, 1, 2):
        wsb = lib.mp_project_fibers_workspace_size(_capi.MP_F32, n, m, q)
        A = Arena([y_h.nbytes, y_h.nbytes, m * 8, m * 8, wsb])
        A.view(0, torch.float32, (n, m)).copy_(torch.from_numpy(y_h))
        A.view(2, torch.float64, (m,)).copy_(torch.from_numpy(O_norms(y_h, q)))
        A.view(3, torch.float64, (m,)).fill_(0.5)
        _capi.check(lib.mp_project_fibers(A.ptr(0), A.ptr(1), _capi.MP_F32, n, m, q, A.ptr(2), A.ptr(3), 0,
                                          A.ptr(4), wsb, torch.cuda.current_stream().cuda_stream))
        A.check_guards()


def O_norms(y, q):
    a = np.abs(y.astype(np.float64))
    return a.sum(0) if q == 0 else (np.sqrt((a * a).sum(0)) if q == 1 else a.max(0))


def test_kernel_attributes_per_device():
    """Function attributes (large dynamic shared memory, non-portable
    clusters) are set per device: the TMA strips, the cluster K2 and the
    euclid sort must launch on a second device of the same process."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs in one process")
    rng = np.random.default_rng(8)
    y_h = rng.normal(size=(3000, 16384)).astype(np.float32)  # 256-thread TMA strips, 16-CTA cluster K2
    eta = 0.05 * float(np.abs(y_h.astype(np.float64)).sum())
    outs = []
    for dev in (0, 1):
        y = torch.from_numpy(y_h).to(f"cuda:{dev}")
        x, b, z = mp.bilevel_project(y, eta, "1", "1")
        xe, be, th = mp.euclid_project_l1inf(y[:, :64].contiguous(), 5.0)
        torch.cuda.synchronize(dev)
        outs.append((x.cpu().numpy(), xe.cpu().numpy()))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
