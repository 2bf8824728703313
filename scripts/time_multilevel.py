"""Device time of mp_multilevel_project for a few specs on a 256^3 tensor."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2405_02086_b200 as mp
from oracle import oracle as O

t_h = np.random.default_rng(4).normal(size=(256, 256, 256)).astype(np.float32)
t = torch.from_numpy(t_h).cuda()
x = torch.empty_like(t)
for spec in ["inf,inf,1", "2,1,1", "1,1,1", "inf,2,1", "1,inf,2", "2,2,inf"]:
    lv = spec.split(",")
    eta = 0.05 * O.multilevel_norm(t_h.astype(np.float64), lv)
    p = mp.MultilevelProjector(t_h.shape, spec, want_chain=False)
    for _ in range(3):
        p(t, x, eta)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        p(t, x, eta)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(spec, round(ms * 1e3, 1), "us", round(2 * t_h.nbytes / (ms * 1e-3) / 1e9), "GB/s (2x tensor)")
