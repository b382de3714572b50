#!/usr/bin/env python
"""Permutation kernel time vs P (graph of 20 launches): one-CTA vs multi-CTA (W4A16_PERMUTE_SINGLE_MAX)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
from paper_2504_16214_b200.moe import ops  # noqa: E402

dev = torch.device("cuda", 0)
for P, E in ((512, 256), (2048, 256), (4096, 256), (8192, 256), (2048, 128), (65536, 256)):
    ids = torch.randint(0, E, (P,), dtype=torch.int32, device=dev)
    ws = torch.empty(max(ops.permute_ws_bytes(P, E), 1), dtype=torch.uint8, device=dev)
    f = lambda: ops.moe_permute(ids, E, ws)  # noqa: E731
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(20):
            f()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    print(f"P={P:6d} E={E}: {a.elapsed_time(b) / 20 * 1e3:7.1f} us")
