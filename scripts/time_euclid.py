"""Device time of the exact Euclidean l1,inf projection (mp_euclid_project)
on config-sized inputs, plus the reference CPU time on the same input
(oracle/_ref, one call) when CPU=1."""
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2405_02086_b200 as mp
from paper_2405_02086_b200 import _build, _capi, datagen

if os.environ.get("MP_B200_LIB"):  # A/B runs: a variant build (scripts/ab_build.sh)
    _build.LIB = os.environ["MP_B200_LIB"]
from oracle import oracle as O

L = _capi.lib()
shapes = [tuple(int(v) for v in s.split("x")) for s in os.environ.get("SHAPES", "10000x10000,4096x16384").split(",")]
rels = [float(r) for r in os.environ.get("RELS", "0.1,0.5").split(",")]
res = []
for (n, m) in shapes:
    y_h = datagen.uniform(2, (n, m), -1.0, 1.0)
    y = torch.from_numpy(y_h).cuda()
    x = torch.empty_like(y)
    wsb = L.mp_euclid_workspace_size(_capi.MP_F32, n, m)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    b = torch.empty(m, dtype=torch.float64, device="cuda")
    info = torch.zeros(C.sizeof(_capi.MpInfo), dtype=torch.uint8, device="cuda")
    nrm = float(np.abs(y_h.astype(np.float64)).max(axis=0).sum())
    for rel in rels:
        eta = rel * nrm
        s = torch.cuda.current_stream()
        call = lambda: _capi.check(L.mp_euclid_project(y.data_ptr(), x.data_ptr(), _capi.MP_F32, n, m, eta,
                                                       b.data_ptr(), info.data_ptr(), 0, ws.data_ptr(), wsb,
                                                       s.cuda_stream))
        for _ in range(3):
            call()
        torch.cuda.synchronize()
        ts = []
        for _ in range(int(os.environ.get("REPS", "10"))):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            call()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        inf = _capi.MpInfo.from_buffer_copy(info.cpu().numpy().tobytes())
        d = {"shape": [n, m], "rel": rel, "ms_median": float(np.median(ts)), "ms_min": float(np.min(ts)),
             "newton_iterations": int(inf.iterations), "theta": inf.tau, "zero_columns": int(inf.zero_columns),
             "workspace_bytes": int(wsb)}
        if os.environ.get("CPU", "0") == "1" and O.ref_available():
            t0 = time.perf_counter()
            xr, br, tr = O.ref_euclid(y_h.astype(np.float64), eta)
            d["cpu_reference_s"] = time.perf_counter() - t0
            d["theta_rel_err"] = abs(inf.tau - tr) / tr if tr else 0.0
            d["budgets_max_rel_err"] = float(np.max(np.abs(b.cpu().numpy() - br) / np.maximum(np.abs(br), 1e-300)))
        print(json.dumps(d), flush=True)
        res.append(d)
