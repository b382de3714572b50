#!/usr/bin/env python
"""One grouped-GEMM launch at DeepSeek-R1 shapes on a chosen number of experts / tokens per expert
(for ncu captures that would be too slow on the full layer). --which gate_up|down."""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402
from paper_2504_16214_b200.moe import ops  # noqa: E402
from paper_2504_16214_b200.moe.weights import random_packed  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--which", default="down")
ap.add_argument("--experts", type=int, default=24)
ap.add_argument("--per-expert", type=int, default=3)
ap.add_argument("--ntok", type=int, default=0)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--sums", type=int, default=1)
a = ap.parse_args()
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
rows = E * a.per_expert
x = (torch.randn((rows, K), device=dev) * 0.5).half()
ntok = a.ntok or ops.pick_ntok(rows * 8, E * 8)
xs = ops.group_sums(x) if a.sums else None
for _ in range(a.reps):
    ops.grouped_gemm(x, w.blocks, E, N // 2 if gated else N, gated, counts, off, ntok, xsum=xs)
torch.cuda.synchronize()
print("ok", a.which, E, a.per_expert, ntok)
