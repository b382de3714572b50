#!/usr/bin/env python
"""Graphed layer time for forced token tiles (16/32/64/128) vs the picked one, per (model, T)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
from paper_2504_16214_b200.moe import moe_w4a16, ops, random_moe_weights, select_experts  # noqa: E402

SHAPES = {"ds": (256, 8, 7168, 2048), "mixtral": (8, 2, 4096, 14336), "qwen3": (128, 8, 2048, 768)}
dev = torch.device("cuda", 0)
for case in sys.argv[1].split(","):
    model, T = case.split(":")
    T = int(T)
    E, K, H, I = SHAPES[model]
    w = random_moe_weights(E, H, I, torch.float16, device=dev, seed=3)
    x = (torch.randn((T, H)) * 0.5).half().to(dev)
    lg = torch.randn((T, E)).to(dev)
    wts, ids = select_experts(lg, K, "softmax", True)
    picked = ops.pick_ntok(T * K, E)
    res = {}
    for nt in (16, 32, 64, 128):
        f = lambda: moe_w4a16(x, w, wts, ids, ntok=nt)  # noqa: E731
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(2):
                f()
        torch.cuda.current_stream().wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            f()
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        res[nt] = round(a.elapsed_time(b) / 20 * 1e3, 1)
        del g
    print(f"{model} T={T} picked {picked}: " + ", ".join(f"ntok {k}: {v} us" for k, v in res.items()), flush=True)
    del w
    torch.cuda.empty_cache()
