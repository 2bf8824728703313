"""One projection of a config-shaped input (for ncu): DT, Q, N, M, REL env."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2405_02086_b200 as mp
from paper_2405_02086_b200 import datagen

dt, q = os.environ.get("DT", "float32"), os.environ.get("Q", "inf")
n, m = int(os.environ.get("N", "4096")), int(os.environ.get("M", "16384"))
y_h = datagen.normal(3, (n, m))
y = torch.from_numpy(y_h).cuda().to(getattr(torch, dt))
x = torch.empty_like(y)
y64 = y_h.astype(np.float64)
nrm = {"1": np.abs(y64).sum(), "2": np.sqrt((y64 * y64).sum(0)).sum(), "inf": np.abs(y64).max(0).sum()}[q]
p = mp.BilevelProjector(n, m, dt, "1", q)
for _ in range(int(os.environ.get("REPS", "2"))):
    p(y, x, float(os.environ.get("REL", "0.05")) * float(nrm))
torch.cuda.synchronize()
inf = p.info()
print("iterations", inf.iterations, "survivors", inf.survivors, "zero_columns", inf.zero_columns)
