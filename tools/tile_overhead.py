#!/usr/bin/env python
"""Per-stage vs per-tile cost of the grouped GEMM: time gate/up-mode and k-pair-mode launches at
several K (stages per tile) with the total weight bytes held ~constant (GPU, CUDA events)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402
from paper_2504_16214_b200.moe import ops  # noqa: E402
from paper_2504_16214_b200.moe.weights import random_packed  # noqa: E402

dev = torch.device("cuda", 0)
gd = torch.Generator(device=dev).manual_seed(1)
TOTAL = 1.6e9  # weight bytes per launch
for gated in (True, False):
    for K in (1024, 2048, 4096, 8192):
        N = 2048 if gated else 7168
        per_e = ops.packed_bytes(1, 2 * N if gated else N, K)
        E = max(1, int(TOTAL // per_e))
        E = min(E, 1024)
        w = random_packed(E, 2 * N if gated else N, K, gated, torch.float16, gd, dev)
        counts = torch.full((E,), 3, dtype=torch.int32, device=dev)
        off = torch.zeros(E + 1, dtype=torch.int32, device=dev)
        off[1:] = torch.cumsum(counts, 0)
        x = (torch.randn((3 * E, K), device=dev) * 0.5).half()
        for _ in range(3):
            ops.grouped_gemm(x, w.blocks, E, N, gated, counts, off, 16)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            ops.grouped_gemm(x, w.blocks, E, N, gated, counts, off, 16)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 10
        byts = E * per_e
        nt = N // 128
        stages_per_tile = K // 128 if gated else K // 256
        tiles = E * nt
        cyc = ms * 1e-3 * 1.965e9
        per_cta_tiles = tiles / 148
        print(f"{'gate_up' if gated else 'down  '} K={K:5d} E={E:4d} tiles={tiles:6d} stages/tile={stages_per_tile:3d} "
              f"ms={ms:.4f} GB/s={byts / ms / 1e6:7.1f} cyc/stage={cyc / (per_cta_tiles * stages_per_tile):6.0f}",
              flush=True)
        del w, x
