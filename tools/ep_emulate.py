#!/usr/bin/env python
"""One rank's expert work of the all-gather EP layer at world size N, emulated on one GPU: the node
batch (N*T tokens, routed over all E experts) through this rank's shard of E/N experts with the
other ranks' ids dropped (-1), exactly the call NcclExchange.experts makes (fp32 partial output).
Prints the graphed time per N next to the single-GPU layer at T tokens.

    python tools/ep_emulate.py [T=64] [N=1,2,4,8]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
from paper_2504_16214_b200.moe import moe_w4a16, ops, random_moe_weights, select_experts  # noqa: E402

E, K, H, I = 256, 8, 7168, 2048
T = int(sys.argv[1]) if len(sys.argv) > 1 else 64
Ns = [int(n) for n in (sys.argv[2] if len(sys.argv) > 2 else "1,2,4,8").split(",")]
dev = torch.device("cuda", 0)
for N in Ns:
    el = E // N
    w = random_moe_weights(el, H, I, torch.float16, device=dev, seed=3)
    x = (torch.randn((N * T, H)) * 0.5).half().to(dev)
    lg = torch.randn((N * T, E)).to(dev)
    wts, ids = select_experts(lg, K, "softmax", True)
    loc = ops.ep_localize(ids, 0, el)  # rank 0's shard
    nt = int(sys.argv[3]) if len(sys.argv) > 3 else ops.pick_ntok(N * T * K // N, el)
    f = lambda: moe_w4a16(x, w, wts, loc, ntok=nt, f32_out=True)  # noqa: E731
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
    local = int((loc >= 0).sum())
    print(f"N={N}: rank shard {el} experts, node batch {N * T} tokens, local pairs {local}, ntok {nt}: "
          f"{a.elapsed_time(b) / 20 * 1e3:.1f} us per step (experts only)", flush=True)
    del w, g
    torch.cuda.empty_cache()
