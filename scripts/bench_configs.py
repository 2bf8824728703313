#!/usr/bin/env python3
"""Device throughput of all five BASELINE.json configs (evidence beside the
headline bench.py line; writes one JSON document to stdout).

Per projection: algorithmic bytes B = 4 * N * (2 + f_surv) (one full read, a
read of the surviving columns, one full write), device time
from external CUDA events around each projection inside a CUDA graph, an L2
read-flush before each projection.  The reference CPU path (oracle/_ref, all
host cores, bench_one recipe) is timed on one call per config.
"""
import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import paper_2405_02086_b200 as mp
from oracle import oracle as O
from paper_2405_02086_b200 import _capi, datagen

REPS = int(os.environ.get("REPS", "10"))
CPU = os.environ.get("CPU", "1") == "1"
lib = _capi.lib()
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(dev)
flush_buf = torch.ones(64 << 20, dtype=torch.float32, device=dev)
workers = os.cpu_count() or 1


def timed_graph(call, nproj=1):
    """Replay a graph of [flush, call] REPS times; device ms per call."""
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    with torch.cuda.stream(stream):
        for e in ev:
            e.record(stream)
        call()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            flush_buf.sum()
            h = (C.c_void_p * 4)(C.c_void_p(ev[0].cuda_event), None, None, C.c_void_p(ev[1].cuda_event))
            lib.mp_profile_events(h, 4)
            call()
            lib.mp_profile_events(None, 0)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        ts = []
        for _ in range(REPS):
            g.replay()
            stream.synchronize()
            ts.append(ev[0].elapsed_time(ev[1]))
    return float(np.median(ts))


def line(name, n_elems, f_surv, ms, cpu_s=None, extra=None, s=4.0):
    b = s * n_elems * (2.0 + f_surv)
    d = {"config": name, "ms": ms, "algo_bytes": b, "GBps": b / (ms * 1e-3) / 1e9, "frac_measured_hbm": b / (ms * 1e-3) / 1e9 / peak,
         "f_surv": f_surv, "elements_per_s": n_elems / (ms * 1e-3)}
    if cpu_s is not None:
        d["cpu_reference_s"] = cpu_s
        d["cpu_reference_GBps"] = b / cpu_s / 1e9
        d["speedup_vs_cpu_reference"] = cpu_s / (ms * 1e-3)
    if extra:
        d.update(extra)
    return d


def cpu_bilevel(y, eta, p, q):
    if not CPU or not O.ref_available():
        return None
    return float(np.median(O.ref_time_bilevel(y, [eta], p, q, reps=1, workers=workers)))


out = {"peak_hbm_gbs": peak, "reps": REPS, "cpu_workers": workers, "results": []}

# config 1
y = datagen.config_input(1)
eta = 0.1 * float(np.abs(y).max(axis=0).astype(np.float64).sum())
yd = torch.from_numpy(y).to(dev)
xd = torch.empty_like(yd)
p = mp.BilevelProjector(*y.shape, device=dev)
ms = timed_graph(lambda: p(yd, xd, eta, stream=stream))
p(yd, xd, eta); torch.cuda.synchronize()
out["results"].append(line("c1 bilevel l1,inf 1000x1000 N(0,1) eta=0.1", y.size, p.info().survivors / y.shape[1], ms,
                           cpu_bilevel(y, eta, "1", "inf"), {"zero_columns": p.info().zero_columns}))

# config 2 (4 radii)
y = datagen.config_input(2)
colmax = np.abs(y).max(axis=0).astype(np.float64)
yd = torch.from_numpy(y).to(dev)
xd = torch.empty_like(yd)
p = mp.BilevelProjector(*y.shape, device=dev)
for rel in (0.001, 0.01, 0.1, 0.5):
    eta = rel * float(colmax.sum())
    ms = timed_graph(lambda: p(yd, xd, eta, stream=stream))
    p(yd, xd, eta); torch.cuda.synchronize()
    out["results"].append(line(f"c2 bilevel l1,inf 10000x10000 U[-1,1] eta={rel}", y.size,
                               p.info().survivors / y.shape[1], ms, cpu_bilevel(y, eta, "1", "inf") if rel in (0.001, 0.5) else None,
                               {"zero_columns": p.info().zero_columns}))
# config 2 in f64 (the C++ drop-in's dtype, the reference's arithmetic)
yd64 = yd.double()
xd64 = torch.empty_like(yd64)
p64 = mp.BilevelProjector(*y.shape, dtype="float64", device=dev)
eta = 0.1 * float(colmax.sum())
ms = timed_graph(lambda: p64(yd64, xd64, eta, stream=stream))
p64(yd64, xd64, eta); torch.cuda.synchronize()
out["results"].append(line("c2 f64 bilevel l1,inf 10000x10000 U[-1,1] eta=0.1", y.size, p64.info().survivors / y.shape[1],
                           ms, None, {"zero_columns": p64.info().zero_columns}, s=8.0))
del yd, xd, yd64, xd64

# config 3 (l1,1 and l1,2)
y = datagen.config_input(3)
yd = torch.from_numpy(y).to(dev)
xd = torch.empty_like(yd)
y64 = y.astype(np.float64)
for q in ("1", "2"):
    eta = 0.05 * (float(np.abs(y64).sum()) if q == "1" else float(np.sqrt((y64 * y64).sum(axis=0)).sum()))
    p = mp.BilevelProjector(*y.shape, q=q, device=dev)
    ms = timed_graph(lambda: p(yd, xd, eta, stream=stream))
    p(yd, xd, eta); torch.cuda.synchronize()
    out["results"].append(line(f"c3 bilevel l1,{q} 4096x16384 N(0,1) eta=0.05", y.size, p.info().survivors / y.shape[1],
                               ms, cpu_bilevel(y, eta, "1", q), {"zero_columns": p.info().zero_columns}))
del yd, xd, y64

# config 4 (tri-level)
t = datagen.config_input(4)
eta = 0.05 * float(np.abs(t).max(axis=0).max(axis=0).astype(np.float64).sum())
td_ = torch.from_numpy(t).to(dev)
xd = torch.empty_like(td_)
mpj = mp.MultilevelProjector(t.shape, "inf,inf,1", device=dev, want_chain=False)
ms = timed_graph(lambda: mpj(td_, xd, eta, stream=stream))
mpj(td_, xd, eta); torch.cuda.synchronize()
cpu_s = None
if CPU and O.ref_available():
    t0 = time.perf_counter()
    O.ref_multilevel(t.astype(np.float64), ["inf", "inf", "1"], eta, workers=workers)
    cpu_s = time.perf_counter() - t0
out["results"].append(line("c4 trilevel l1,inf,inf 256^3 N(0,1) eta=0.05", t.size, mpj.info().survivors / t.shape[2], ms,
                           cpu_s))
del td_, xd

# exact Euclidean l1,inf at the config-1 and config-3 shapes
for cfg, rel in ((1, 0.1), (3, 0.1)):
    y = datagen.config_input(cfg)
    n_, m_ = y.shape
    eta = rel * float(np.abs(y).max(axis=0).astype(np.float64).sum())
    yd = torch.from_numpy(y).to(dev)
    xd = torch.empty_like(yd)
    wsb = lib.mp_euclid_workspace_size(_capi.MP_F32, n_, m_)
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    bd = torch.empty(m_, dtype=torch.float64, device=dev)
    info = torch.zeros(C.sizeof(_capi.MpInfo), dtype=torch.uint8, device=dev)
    call = lambda: _capi.check(lib.mp_euclid_project(yd.data_ptr(), xd.data_ptr(), _capi.MP_F32, n_, m_, eta,
                                                     bd.data_ptr(), info.data_ptr(), 0, ws.data_ptr(), wsb,
                                                     stream.cuda_stream))
    ms = timed_graph(call)
    inf = _capi.MpInfo.from_buffer_copy(info.cpu().numpy().tobytes())
    cpu_s = None
    if CPU and O.ref_available() and cfg == 1:
        t0 = time.perf_counter()
        O.ref_euclid(y.astype(np.float64), eta)
        cpu_s = time.perf_counter() - t0
    out["results"].append(line(f"euclid l1,inf {n_}x{m_} (config-{cfg} input) eta={rel}", y.size, 1.0, ms, cpu_s,
                               {"newton_iterations": int(inf.iterations), "theta": inf.tau,
                                "note": "algorithmic bytes as a bi-level projection (read + write); the sort "
                                        "dominates, not HBM"}))
    del yd, xd, ws

# config 5 (loop of 100: perturb + project)
y = datagen.config_input(5)
eta = datagen.config5_eta(np.abs(y).max(axis=0).astype(np.float64))
xd = torch.from_numpy(y).to(dev)
p = mp.BilevelProjector(*y.shape, device=dev)
ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(100)]
pv = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(100)]
zeros = []
with torch.cuda.stream(stream):
    for row in ev:
        for e in row:
            e.record(stream)  # torch must see a record before elapsed_time
    for it in range(100):
        pv[it][0].record(stream)
        if it > 0:
            mp.perturb_gaussian(xd, 1e-4, seed=6, iteration=it, stream=stream)
        pv[it][1].record(stream)
        h = (C.c_void_p * 4)(C.c_void_p(ev[it][0].cuda_event), None, None, C.c_void_p(ev[it][1].cuda_event))
        lib.mp_profile_events(h, 4)
        p(xd, xd, eta, stream=stream)
        lib.mp_profile_events(None, 0)
        stream.synchronize()
        zeros.append(int(p.info().zero_columns))
proj_ms = [ev[i][0].elapsed_time(ev[i][1]) for i in range(100)]
pert_ms = [pv[i][0].elapsed_time(pv[i][1]) for i in range(1, 100)]
m = y.shape[1]
bytes_tot = sum(4.0 * y.size * (2.0 + (m - z) / m) for z in zeros)
cpu_s = cpu_bilevel(y, eta, "1", "inf")
out["results"].append({"config": "c5 loop: 100 x (perturb N(0,1e-4^2) + bilevel l1,inf) 32768x8192 Laplace(0,0.01)",
                       "projection_ms_total": sum(proj_ms), "projection_ms_median": float(np.median(proj_ms)),
                       "GBps": bytes_tot / (sum(proj_ms) * 1e-3) / 1e9,
                       "frac_measured_hbm": bytes_tot / (sum(proj_ms) * 1e-3) / 1e9 / peak,
                       "perturb_ms_median": float(np.median(pert_ms)),
                       "perturb_GBps": 8.0 * y.size / (np.median(pert_ms) * 1e-3) / 1e9,
                       "zero_columns_first_last": [zeros[0], zeros[1], zeros[49], zeros[-1]],
                       "zeroed_fraction_by_iteration": [z / m for z in zeros[:6]] + [zeros[-1] / m],
                       "cpu_reference_s_iter0": cpu_s,
                       "note": "eager loop (no L2 flush: the perturbation streams the whole matrix between calls)"})
print(json.dumps(out, indent=1))
