"""One config-3 l_{1,1} projection (4096 x 16384 N(0,1), eta = 0.05 ||Y||_{1,1}) through the C-ABI."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2405_02086_b200 as mp
from paper_2405_02086_b200 import _build, datagen

if os.environ.get("MP_B200_LIB"):
    _build.LIB = os.environ["MP_B200_LIB"]

q = os.environ.get("Q", "1")
y_h = datagen.config_input(3)
eta = 0.05 * float(np.abs(y_h).astype(np.float64).sum()) if q == "1" else 0.05 * float(
    np.sqrt((y_h.astype(np.float64) ** 2).sum(axis=0)).sum())
y = torch.from_numpy(y_h).cuda()
x = torch.empty_like(y)
p = mp.BilevelProjector(4096, 16384, "float32", "1", q)
for _ in range(int(os.environ.get("REPS", "2"))):
    p(y, x, eta)
torch.cuda.synchronize()
print(p.info().iterations, p.info().survivors)
