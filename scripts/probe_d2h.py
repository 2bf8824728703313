"""PCIe probe: pinned D2H / H2D bandwidth, one vs two streams (e2e ceiling)."""
import time
import torch
n = 100_000_000
d = torch.ones(n, device="cuda")
hs = [torch.empty(n, pin_memory=True) for _ in range(2)]
s = [torch.cuda.Stream() for _ in range(4)]
def bw(fn, reps=10):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps
def one():
    hs[0].copy_(d, non_blocking=True)
def two():
    with torch.cuda.stream(s[0]): hs[0][: n // 2].copy_(d[: n // 2], non_blocking=True)
    with torch.cuda.stream(s[1]): hs[0][n // 2:].copy_(d[n // 2:], non_blocking=True)
def four():
    q = n // 4
    for i in range(4):
        with torch.cuda.stream(s[i]): hs[0][i*q:(i+1)*q].copy_(d[i*q:(i+1)*q], non_blocking=True)
def h2d():
    d.copy_(hs[1], non_blocking=True)
def both():
    with torch.cuda.stream(s[0]): hs[0].copy_(d, non_blocking=True)
    with torch.cuda.stream(s[1]): d2.copy_(hs[1], non_blocking=True)
d2 = torch.empty_like(d)
for name, fn in [("d2h 1 stream", one), ("d2h 2 streams", two), ("d2h 4 streams", four), ("h2d", h2d), ("d2h+h2d", both)]:
    t = bw(fn)
    print(f"{name}: {4 * n / t / 1e9:.1f} GB/s per direction-call ({t*1e3:.2f} ms)")
