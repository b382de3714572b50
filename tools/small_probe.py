#!/usr/bin/env python
"""Eager layer steps for launch-list profiling of small batches (ncu --metrics gpu__time_duration.sum):
each (model, T) runs `--reps` steps; an NVTX-free marker kernel (torch.cuda._sleep) separates cases.

    ncu --metrics gpu__time_duration.sum --csv --log-file out.csv python tools/small_probe.py ds:1,ds:16,qwen3:256
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
SHAPES = {"ds": (256, 8, 7168, 2048), "mixtral": (8, 2, 4096, 14336), "qwen3": (128, 8, 2048, 768)}


def main():
    import torch
    from paper_2504_16214_b200.moe import fused_moe_w4a16, random_moe_weights, w4a16_linear
    from paper_2504_16214_b200.moe.weights import random_packed
    dev = torch.device("cuda", 0)
    reps = 2
    cache = {}
    for case in sys.argv[1].split(","):
        model, T = case.split(":")
        T = int(T)
        if model == "llama":
            w = cache.setdefault(model, random_packed(1, 14336, 4096, False, torch.float16, 3, dev))
            x = (torch.randn((T, 4096), device=dev) * 0.5).half()
            for _ in range(reps):
                w4a16_linear(x, w)
        else:
            E, k, H, I = SHAPES[model]
            w = cache.setdefault(model, random_moe_weights(E, H, I, torch.float16, device=dev, seed=5))
            x = (torch.randn((T, H), device=dev) * 0.5).half()
            lg = torch.randn((T, E), device=dev)
            for _ in range(reps):
                fused_moe_w4a16(x, lg, w, k, "softmax", True)
        torch.cuda.synchronize()
        torch.cuda._sleep(1000)
        torch.cuda.synchronize()
        print("done", case, flush=True)


if __name__ == "__main__":
    main()
