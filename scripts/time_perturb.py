import os, sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch, ctypes as C
from paper_2405_02086_b200 import _build, _capi
if os.environ.get("MP_B200_LIB"): _build.LIB = os.environ["MP_B200_LIB"]
L = _capi.lib()
x = torch.randn(32768, 8192, device="cuda")
s = torch.cuda.current_stream()
ts = []
for i in range(12):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); L.mp_perturb_gaussian(x.data_ptr(), _capi.MP_F32, x.numel(), C.c_double(1e-4), C.c_uint64(7), C.c_uint64(i), C.c_void_p(s.cuda_stream)); e1.record()
    torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
print(os.environ.get("MP_B200_LIB", "base")[-12:], "perturb 1 GiB: median %.1f us" % (1e3 * float(np.median(ts[2:]))))
