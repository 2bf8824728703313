import ctypes as C, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2405_02086_b200 as mp
from paper_2405_02086_b200 import _capi
lib = _capi.lib()
y = torch.randn(4000, 4000, device="cuda"); x = torch.empty_like(y)
p = mp.BilevelProjector(4000, 4000)
s = torch.cuda.Stream()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
with torch.cuda.stream(s):
    for e in ev: e.record(s)
    h = (C.c_void_p * 4)(*[C.c_void_p(e.cuda_event) for e in ev])
    lib.mp_profile_events(h, 4)
    p(y, x, 100.0, stream=s)
    lib.mp_profile_events(None, 0)
torch.cuda.synchronize()
try:
    print("eager lib-recorded:", [ev[0].elapsed_time(e) for e in ev[1:]])
except Exception as ex:
    print("eager lib-recorded FAILED", ex)
ev2 = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    with torch.cuda.graph(g, stream=s):
        ev2[0].record(s); p(y, x, 100.0, stream=s); ev2[1].record(s)
g.replay(); torch.cuda.synchronize()
try:
    print("graph torch-recorded:", ev2[0].elapsed_time(ev2[1]))
except Exception as ex:
    print("graph torch-recorded FAILED", ex)
