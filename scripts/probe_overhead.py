"""Fixed overheads around one projection graph: empty-ish graphs timed the way bench.py times a projection."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
torch.cuda.set_device(0)
s = torch.cuda.Stream()
buf = torch.zeros(10000, dtype=torch.int64, device="cuda")
big = torch.zeros(1 << 20, dtype=torch.float32, device="cuda")
flush_buf = torch.ones(64 << 20, dtype=torch.float32, device="cuda")

def timeit(fn, label):
    with torch.cuda.stream(s):
        fn(); torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            fn()
        ts = []
        for _ in range(30):
            flush_buf.sum()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s); g.replay(); b.record(s)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    print(f"{label:40s} median {ts[len(ts)//2]:.2f} us  min {ts[0]:.2f}")

timeit(lambda: buf.zero_(), "memset-kernel (torch zero_ 80KB)")
timeit(lambda: torch.cuda.current_stream().wait_stream(s) or buf.fill_(0), "fill kernel")
def memset_api():
    import ctypes
    cudart = ctypes.CDLL("libcudart.so.12") if False else None
timeit(lambda: (big.mul_(1.0)), "tiny elementwise 4MB")
timeit(lambda: (buf.zero_(), big.mul_(1.0)), "2 kernels")
