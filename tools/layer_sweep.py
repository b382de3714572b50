#!/usr/bin/env python
"""Whole-layer time (CUDA graph, FusedMoEGraph) across token counts for the BASELINE model shapes.
Prints one line per (model, T): ms, algorithmic GB/s and TFLOP/s, fractions of the measured peaks.

    python tools/layer_sweep.py [--model ds,mixtral,qwen3] [--tokens 1,4,16,64,256]
"""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

SHAPES = {"ds": (256, 8, 7168, 2048), "mixtral": (8, 2, 4096, 14336), "qwen3": (128, 8, 2048, 768)}


def main():
    import torch
    from bench import layer_bytes, layer_flops, peaks
    from paper_2504_16214_b200.moe import FusedMoEGraph, random_moe_weights, select_experts
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="ds,mixtral,qwen3")
    ap.add_argument("--tokens", default="1,4,16,64,256,1024")
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    hbm, tc, tcs, _ = peaks()
    dev = torch.device("cuda", 0)
    for model in a.model.split(","):
        E, k, H, I = SHAPES[model]
        w = random_moe_weights(E, H, I, torch.float16, device=dev, seed=5)
        g = torch.Generator().manual_seed(0)
        for T in map(int, a.tokens.split(",")):
            x = (torch.randn((T, H), generator=g) * 0.5).half().to(dev)
            lg = torch.randn((T, E), generator=g).to(dev)
            _, ids = select_experts(lg, k, "softmax", True)
            et = int(torch.unique(ids).numel())
            gr = FusedMoEGraph(w, T, k, "softmax", True, torch.float16, dev)
            gr(x, lg)
            for _ in range(3):
                gr()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.reps):
                gr()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.reps
            by, fl = layer_bytes(et, T, H, I, k), layer_flops(T, k, H, I)
            print(json.dumps({"model": model, "T": T, "experts_touched": et, "ms": round(ms, 4),
                              "GB/s": round(by / ms / 1e6, 1), "hbm_frac": round(by / ms / 1e6 / hbm, 4),
                              "TFLOP/s": round(fl / ms / 1e9, 2), "tc_frac": round(fl / ms / 1e9 / tc, 4)}),
                  flush=True)
            del gr
        del w
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
