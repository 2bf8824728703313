"""Small invocations of every kernel family (for compute-sanitizer memcheck /
racecheck / synccheck runs): bi-level (all p, q; f32, f64; K3b routes),
multi-level, vector balls, aggregate, fibers, euclid, perturbation, async
sweep."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2405_02086_b200 as mp
from paper_2405_02086_b200 import _capi

rng = np.random.default_rng(0)
# l1 inner strips on every route: 64 / 128 / 256-thread TMA strips and the
# mbarrier ring (600, 1500, 3000 rows), hybrid cp.async strips (4096 f32),
# 512-thread TMA strips (f64 4097..8192), register strips, shared quads
for dt in (np.float32, np.float64):
    for shape in [(600, 24), (1500, 16), (3000, 8), (4096, 16), (4100, 8), (200, 32)]:
        y = rng.normal(size=shape).astype(dt)
        mp.bilevel_project(y, 0.05 * float(np.abs(y.astype(np.float64)).sum()), "1", "1")
# K2 on a DSMEM cluster (m > 12288) and on the cooperative grid (m > 98304)
for m in (20000, 100003):
    y = rng.uniform(-1, 1, size=(3, m)).astype(np.float32)
    for q in ("inf", "1"):
        mp.bilevel_project(y, 0.1 * float(np.abs(y).max(axis=0).sum()), "1", q)
for dt in (np.float32, np.float64):
    for shape in [(37, 45), (300, 64), (9000, 8), (5, 3)]:
        y = rng.normal(size=shape).astype(dt)
        for p in ("1", "2", "inf"):
            for q in ("1", "2", "inf"):
                eta = 0.2 * float(np.abs(y).max(axis=0).sum())
                mp.bilevel_project(y, eta, p, q)
    t = rng.normal(size=(6, 7, 8)).astype(dt)
    mp.multilevel_project(t, "inf,inf,1", 0.3)
    mp.multilevel_project(t, "2,1,inf", 0.3)
    mp.multilevel_project(rng.normal(size=(4, 5, 6, 7)).astype(dt), "1,2,inf,1", 0.3)
    mp.project_ball(rng.normal(size=1000).astype(dt), "1", 3.0)
    mp.euclid_project_l1inf(rng.normal(size=(100, 40)).astype(dt), 5.0)
yt = torch.from_numpy(rng.normal(size=(200, 96)).astype(np.float32)).cuda()
proj = mp.BilevelProjector(200, 96, "float32", "1", "1")
proj(yt, torch.empty_like(yt), 10.0)
mp.perturb_gaussian(yt, 1e-3, seed=1, iteration=2)
mp.bilevel_radius_sweep(rng.normal(size=(64, 33)).astype(np.float32), [0.1, 1.0, 5.0])
torch.cuda.synchronize()
print("sanitize cases done")
