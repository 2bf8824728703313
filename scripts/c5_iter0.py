import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2405_02086_b200 as mp
from paper_2405_02086_b200 import datagen
y = datagen.config_input(5)
eta = datagen.config5_eta(np.abs(y).max(axis=0).astype(np.float64))
yd = torch.from_numpy(y).cuda(); xd = torch.empty_like(yd)
p = mp.BilevelProjector(*y.shape)
flush = torch.ones(64 << 20, device="cuda")
ts = []
for r in range(12):
    flush.sum()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); p(yd, xd, eta); e1.record(); torch.cuda.synchronize()
    if r >= 2: ts.append(e0.elapsed_time(e1))
print("c5 iter0 zero_columns", p.info().zero_columns, "ms", np.median(ts))
