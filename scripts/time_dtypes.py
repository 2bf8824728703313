import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2405_02086_b200 as mp
from paper_2405_02086_b200 import datagen
y = datagen.config_input(3)
for dt in ("float32", "float64"):
    yd = torch.from_numpy(y).cuda().to(getattr(torch, dt))
    xd = torch.empty_like(yd)
    for q in ("1", "2", "inf"):
        y64 = y.astype(np.float64)
        eta = 0.05 * (float(np.abs(y64).sum()) if q == "1" else float(np.sqrt((y64*y64).sum(0)).sum()) if q == "2" else float(np.abs(y64).max(0).sum()))
        p = mp.BilevelProjector(*y.shape, dtype=dt, q=q)
        for _ in range(3): p(yd, xd, eta)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10): p(yd, xd, eta)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        s = 4 if dt == "float32" else 8
        print(dt, q, round(ms * 1e3, 1), "us", round(s * y.size * 2 / (ms * 1e-3) / 1e9), "GB/s")
