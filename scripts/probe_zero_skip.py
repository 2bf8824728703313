"""K3 zero-budget read skipping: L2 read sectors of mp_project_fibers (l_inf)
with all / 90% random / no columns at budget 0 (run under ncu)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2405_02086_b200 import _capi

L = _capi.lib()
n, m = 32768, 8192
y = torch.randn(n, m, device="cuda")
x = torch.empty_like(y)
v = y.abs().amax(0).double()
ws = torch.empty(max(L.mp_project_fibers_workspace_size(_capi.MP_F32, n, m, 2), 256), dtype=torch.uint8,
                 device="cuda")
rng = np.random.default_rng(0)
MODE = int(os.environ.get("LDMODE", "0"))
for name, live in [("rand10", rng.random(m) < 0.1), ("all_live", np.ones(m, bool))]:
    u = torch.from_numpy(np.where(live, 0.5, 0.0)).cuda()
    ts = []
    for _ in range(int(os.environ.get("REPS", "2"))):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        _capi.check(L.mp_project_fibers(y.data_ptr(), x.data_ptr(), _capi.MP_F32, n, m, 2, v.data_ptr(), u.data_ptr(),
                                        MODE << 8, ws.data_ptr(), ws.numel(), torch.cuda.current_stream().cuda_stream))
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(name, "mode", MODE, "live fraction", live.mean(), "median ms", np.median(ts[1:] or ts))
