"""Device-side timeline of one config-2 projection (graph replay, L2 flushed
before), from the kernels' own %globaltimer marks (mp_profile_timeline)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2405_02086_b200 as mp
from paper_2405_02086_b200 import _build, _capi, datagen

if os.environ.get("MP_B200_LIB"):  # A/B runs: a variant build (scripts/ab_build.sh)
    _build.LIB = os.environ["MP_B200_LIB"]

L = _capi.lib()
torch.cuda.set_device(0)
n = int(os.environ.get("N", "10000"))
m = int(os.environ.get("M", str(n)))
q = os.environ.get("Q", "inf")
y_h = datagen.normal(3, (n, m)) if os.environ.get("DIST") == "normal" else datagen.uniform(2, (n, m), -1.0, 1.0)
DT = os.environ.get("DT", "float32")
y = torch.from_numpy(y_h).cuda().to(getattr(torch, DT))
x = torch.empty_like(y)
colmax = np.abs(y_h).max(axis=0).astype(np.float64)
p = mp.BilevelProjector(n, m, DT, "1", q)
flush_buf = torch.ones(64 << 20, dtype=torch.float32, device="cuda")
tl = torch.empty(16, dtype=torch.int64, device="cuda")
s = torch.cuda.Stream()
for rel in [float(r) for r in os.environ.get("RELS", "0.001,0.5").split(",")]:
    eta = rel * float(colmax.sum()) if q == "inf" else rel * float(np.abs(y_h).astype(np.float64).sum())
    with torch.cuda.stream(s):
        p(y, x, eta, stream=s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            p(y, x, eta, stream=s)
    res = []
    for rep in range(20):
        init = torch.tensor([2**63 - 1, 0] * 4 + [0] * 8, dtype=torch.int64, device="cuda")
        tl.copy_(init)
        L.mp_profile_timeline(tl.data_ptr())
        with torch.cuda.stream(s):
            flush_buf.sum()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            g.replay()
            e1.record(s)
        torch.cuda.synchronize()
        L.mp_profile_timeline(None)
        t = tl.cpu().numpy().astype(np.float64)
        t0 = t[0]
        rel_t = [(t[i] - t0) / 1e3 if t[i] not in (0, 2**63 - 1) else float("nan") for i in range(8)]
        res.append(rel_t + [e0.elapsed_time(e1) * 1e3])
        extra = t[8:16]
    if extra[2] > 0:
        print(f"  l1: mean passes {extra[0] / extra[2]:.2f} per strip ({extra[3] / extra[2]:.2f} exact) over"
              f" {extra[2]:.0f} strips; max per CTA {extra[1]:.0f}")
        tot = extra[4] + extra[5] + extra[6]
        if tot > 0:
            print(f"  l1 CTA cycles: wait-for-strip {extra[4] / tot:.1%}  passes {extra[5] / tot:.1%}  "
                  f"apply {extra[6] / tot:.1%}  (per strip: {extra[4] / extra[2]:.0f} / {extra[5] / extra[2]:.0f} / "
                  f"{extra[6] / extra[2]:.0f} cycles; apply until the stores are issued {extra[7] / extra[2]:.0f})")
    inf_ = p.info()
    print(f"  info: iterations={inf_.iterations} survivors={inf_.survivors} zero_columns={inf_.zero_columns}")
    r = np.median(np.array(res), axis=0)
    print(f"rel={rel}: event total {r[8]:.1f} us | K1 {r[0]:.1f}->{r[1]:.1f}  fin {r[2]:.1f}->{r[3]:.1f}  "
          f"K2 {r[4]:.1f}->{r[5]:.1f}  K3 {r[6]:.1f}->{r[7]:.1f}")
    print(f"   gaps: K1end->K2start {r[4]-r[1]:.1f}  K2 {r[5]-r[4]:.1f}  K2end->K3start(any) {r[6]-r[5]:.1f}  "
          f"K3 span {r[7]-r[6]:.1f}")
