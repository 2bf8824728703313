"""Time the outer projection (K2) alone: mp_project_ball on f64 vectors of
several lengths, 200 back-to-back calls in one CUDA graph."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2405_02086_b200 import _capi

L = _capi.lib()
torch.cuda.set_device(0)
s = torch.cuda.Stream()
for n in [16, 1024, 4096, 10000, 12288, 12289, 20000, 50000, 98304, 200000]:
    for q in (0, 2):
        y = torch.rand(n, dtype=torch.float64, device="cuda") + 0.5
        x = torch.empty_like(y)
        ws = torch.zeros(L.mp_project_ball_workspace_size(1, n, q), dtype=torch.uint8, device="cuda")
        info = torch.zeros(64, dtype=torch.uint8, device="cuda")
        r = float(y.sum()) * 0.01 if q == 0 else 0.5

        def call():
            _capi.check(L.mp_project_ball(y.data_ptr(), x.data_ptr(), 1, n, q, r, info.data_ptr(), ws.data_ptr(),
                                          ws.numel(), s.cuda_stream))
        with torch.cuda.stream(s):
            call()
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for _ in range(200):
                    call()
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            g.replay()
            e1.record(s)
        torch.cuda.synchronize()
        print(f"n={n:7d} q={q} {e0.elapsed_time(e1) / 200 * 1e3:8.2f} us/call")
