#!/usr/bin/env python
"""Fixed cost of one grouped-GEMM launch: a CUDA graph of 20 back-to-back launches with tiny work
(1 expert, 1 row) against real work, Qwen3 / DS-R1 shapes (GPU)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
from paper_2504_16214_b200.moe import ops  # noqa: E402
from paper_2504_16214_b200.moe.weights import random_packed  # noqa: E402

dev = torch.device("cuda", 0)
gd = torch.Generator(device=dev).manual_seed(1)


def run(E, rows_per, N, K, gated, ntok=16, n=20):
    w = random_packed(E, 2 * N if gated else N, K, gated, torch.float16, gd, dev)
    counts = torch.full((E,), rows_per, dtype=torch.int32, device=dev)
    off = torch.zeros(E + 1, dtype=torch.int32, device=dev)
    off[1:] = torch.cumsum(counts, 0)
    x = (torch.randn((E * rows_per, K), device=dev) * 0.5).half()
    xs = ops.group_sums(x) if ntok <= 16 else None
    out = torch.empty((E * rows_per, N), dtype=torch.float16, device=dev)
    f = lambda: ops.grouped_gemm(x, w.blocks, E, N, gated, counts, off, ntok, out=out, xsum=xs)  # noqa: E731
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(n):
            f()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / n * 1e3
    wb = E * ops.packed_bytes(1, 2 * N if gated else N, K)
    print(f"E={E:3d} rows/expert={rows_per} N={N} K={K} gated={gated}: {us:7.1f} us/launch, {wb / us / 1e3:7.1f} GB/s weights")


run(1, 1, 768, 2048, True)     # qwen3 gate/up, 1 expert (6 tiles)
run(1, 1, 2048, 768, False)    # qwen3 down, 1 expert
run(88, 1, 768, 2048, True)    # qwen3 T=16-like
run(88, 1, 2048, 768, False)
run(8, 1, 2048, 7168, True)    # DS T=1
run(8, 1, 7168, 2048, False)
