"""Copy ceiling at the headline size: torch device-to-device copies of 400 MB
(and 2 GB, the MEASURED_PEAKS size) after an L2 flush, CUDA events."""
import torch
flush = torch.ones(64 << 20, device="cuda")
for nbytes in (400_000_000, 800_000_000, 2_000_000_000):
    n = nbytes // 4
    a = torch.ones(n, device="cuda")
    b = torch.empty_like(a)
    ts = []
    for rep in range(12):
        flush.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); b.copy_(a); e1.record()
        torch.cuda.synchronize()
        if rep >= 2:
            ts.append(e0.elapsed_time(e1))
    ts.sort()
    t = ts[len(ts) // 2]
    print(f"copy {nbytes/1e6:.0f} MB -> {nbytes/1e6:.0f} MB: median {t*1e3:.1f} us = {2*nbytes/t/1e6:.0f} GB/s (best {2*nbytes/ts[0]/1e6:.0f})")
