#!/usr/bin/env python
"""Stream-K vs split-K / whole tiles on single decode GEMMs (graphed, back-to-back replays):
Llama-3-8B dense M=1, DS-R1 T=1 gate/up and down (8 experts x 1 row), Mixtral T=1. The library
reads W4A16_STREAMK / W4A16_SK_LMIN / W4A16_SK_FIX per call, so one process sweeps them."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2504_16214_b200.moe import ops  # noqa: E402
from paper_2504_16214_b200.moe.weights import random_packed  # noqa: E402

dev = torch.device("cuda", 0)


def timed(fn, reps=200):
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        fn()
    torch.cuda.current_stream().wait_stream(side)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    for _ in range(20):
        g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(3):
        a.record()
        for _ in range(reps):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / reps * 1e3)
    return best


cases = {
    "llama_M1": (1, 14336, 4096, False),
    "ds_gate_up_T1": (8, 2048, 7168, True),
    "ds_down_T1": (8, 7168, 2048, False),
    "mixtral_gate_up_T1": (2, 14336, 4096, True),
    "mixtral_down_T1": (2, 4096, 14336, False),
}
settings = [("off", {"W4A16_STREAMK": "0"}), ("sk", {"W4A16_STREAMK": "1"}),
            ("sk_fix8", {"W4A16_STREAMK": "1", "W4A16_SK_FIX": "8"}),
            ("sk_lmin8", {"W4A16_STREAMK": "1", "W4A16_SK_LMIN": "8"})]
for name, (E, N, K, gated) in cases.items():
    w = random_packed(E, 2 * N if gated else N, K, gated, torch.float16, 3, dev)
    counts = torch.ones(E, dtype=torch.int32, device=dev)
    off = torch.arange(E + 1, dtype=torch.int32, device=dev)
    x = (torch.randn((E, K), device=dev) * 0.5).half()
    xs = ops.group_sums(x)
    out = torch.empty((E, N), dtype=torch.float16, device=dev)
    res = []
    for tag, env in settings:
        for k in ("W4A16_STREAMK", "W4A16_SK_FIX", "W4A16_SK_LMIN"):
            os.environ.pop(k, None)
        os.environ.update(env)
        ws = torch.zeros(max(ops.gemm_ws_bytes(E, K, E, N, gated, 16), 1), dtype=torch.uint8, device=dev)
        us = timed(lambda: ops.grouped_gemm(x, w.blocks, E, N, gated, counts, off, 16, out=out, xsum=xs, workspace=ws))
        res.append(f"{tag} {us:6.1f}")
    print(f"{name:20s}", " | ".join(res), flush=True)
