#!/usr/bin/env python
"""SM clock and power while one grouped GEMM runs back to back for ~3 s (is a prefill kernel power-
capped?). Also reports the kernel's TFLOP/s and, with --trace, clock64 vs globaltimer of CTA 0."""
import argparse
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402
from paper_2504_16214_b200.moe import ops  # noqa: E402
from paper_2504_16214_b200.moe.weights import random_packed  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--which", default="gate_up")
ap.add_argument("--experts", type=int, default=64)
ap.add_argument("--per-expert", type=int, default=256)
ap.add_argument("--ntok", type=int, default=128)
ap.add_argument("--seconds", type=float, default=3.0)
a = ap.parse_args()
import pynvml  # noqa: E402
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
H, I = 7168, 2048
dev = torch.device("cuda", 0)
E = a.experts
gd = torch.Generator(device=dev).manual_seed(1)
gated = a.which == "gate_up"
N, K = (2 * I, H) if gated else (H, I)
w = random_packed(E, N, K, gated, torch.float16, gd, dev)
counts = torch.full((E,), a.per_expert, dtype=torch.int32, device=dev)
off = torch.zeros(E + 1, dtype=torch.int32, device=dev)
off[1:] = torch.cumsum(counts, 0)
x = (torch.randn((E * a.per_expert, K), device=dev) * 0.5).half()
nout = N // 2 if gated else N
out = torch.empty((E * a.per_expert, nout), dtype=torch.float16, device=dev)
for _ in range(3):
    ops.grouped_gemm(x, w.blocks, E, nout, gated, counts, off, a.ntok, out=out)
torch.cuda.synchronize()
samples, stop = [], threading.Event()


def sampler():
    while not stop.is_set():
        samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                        pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
        stop.wait(0.01)


t = threading.Thread(target=sampler, daemon=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 0
t.start()
t0 = time.time()
e0.record()
while time.time() - t0 < a.seconds:
    for _ in range(10):
        ops.grouped_gemm(x, w.blocks, E, nout, gated, counts, off, a.ntok, out=out)
        n += 1
    torch.cuda.synchronize()
e1.record()
torch.cuda.synchronize()
stop.set()
t.join()
ms = e0.elapsed_time(e1) / n
flops = 2.0 * E * a.per_expert * N * K
mhz = sorted(s[0] for s in samples)
pw = sorted(s[1] for s in samples)
rs = 0
for s in samples:
    rs |= s[2]
print(f"{a.which} E={E} rows/expert={a.per_expert}: {ms:.3f} ms/launch, {flops / ms / 1e9:.1f} TFLOP/s; "
      f"SM clock median {mhz[len(mhz) // 2]} MHz (min {mhz[0]}, max {mhz[-1]}), power median {pw[len(pw) // 2]:.0f} W "
      f"max {pw[-1]:.0f} W, reasons mask {rs:#x}, samples {len(samples)}")
