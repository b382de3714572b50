#!/usr/bin/env python
"""Read-only HBM bandwidth ceiling (the decode GEMMs only read): torch reductions over a 4 GiB
buffer, against the read+write copy figure MEASURED_PEAKS.json quotes. CUDA events, best of 10."""
import torch

dev = torch.device("cuda", 0)
n = 4 << 30
buf = torch.empty(n, dtype=torch.uint8, device=dev)
buf.random_(0, 255)


def best(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) / 1e3)
    return min(ts)


for name, view in (("sum int32", buf.view(torch.int32)), ("sum bf16->f32", buf.view(torch.bfloat16)),
                   ("amax f32", buf.view(torch.float32))):
    if "amax" in name:
        t = best(lambda: view.amax())
    elif "bf16" in name:
        t = best(lambda: view.sum(dtype=torch.float32))
    else:
        t = best(lambda: view.sum(dtype=torch.int64))
    print(f"{name:16s} read {n / t / 1e9:8.1f} GB/s")
half = buf[: n // 2]
t = best(lambda: buf[n // 2:].copy_(half))
print(f"{'copy':16s} r+w  {n / t / 1e9:8.1f} GB/s")
