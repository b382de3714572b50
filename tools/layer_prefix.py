#!/usr/bin/env python
"""Incremental cost of each kernel of the single-GPU layer as the graph actually runs it (PDL,
back-to-back replays): graphs of growing prefixes of the decode layer path at a given model / T.

    python tools/layer_prefix.py ds 1 [ds 16 qwen3 256 ...]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
from paper_2504_16214_b200.moe import ops, random_moe_weights  # noqa: E402

SHAPES = {"ds": (256, 8, 7168, 2048), "mixtral": (8, 2, 4096, 14336), "qwen3": (128, 8, 2048, 768)}
dev = torch.device("cuda", 0)


def run(model, T):
    E, K, H, I = SHAPES[model]
    w = random_moe_weights(E, H, I, torch.float16, device=dev, seed=7)
    x = (torch.randn((T, H)) * 0.5).half().cuda()
    lg = torch.randn((T, E)).cuda()
    P = T * K
    nt = ops.pick_ntok(P, E)
    decode = nt <= 16
    perm_ws = torch.empty(max(ops.permute_ws_bytes(P, E), 1), dtype=torch.uint8, device=dev)
    xp = torch.empty((P, H), dtype=torch.float16, device=dev)
    xs = torch.empty(ops.sums_shape(P, H), dtype=torch.float32, device=dev)
    hbuf = torch.empty((P, I), dtype=torch.float16, device=dev)
    hs = torch.empty(ops.sums_shape(P, I), dtype=torch.float32, device=dev)
    yp = torch.empty((P, H), dtype=torch.float16, device=dev)
    gws = [torch.zeros(max(ops.gemm_ws_bytes(P, k_, E, n_, g_, nt), 1), dtype=torch.uint8, device=dev)
           for k_, n_, g_ in ((H, I, True), (I, H, False))]
    small = P <= 64
    stages = ["route+permute", "gather", "gate_up", "down", "combine"]

    def layer(upto):
        if small:
            ids, wts, counts, offsets, sp, pp = ops.route_permute(lg, K, "softmax", True)
        else:
            ids, wts = ops.route_topk(lg, K, "softmax", True)
            counts, offsets, sp, pp = ops.moe_permute(ids, E, perm_ws)
        if upto == 0:
            return
        if decode:
            ops.moe_gather_sums(x, sp, K, P, offsets[E:], out=xp, sums=xs)
        else:
            ops.moe_gather(x, sp, K, P, offsets[E:], out=xp)
        if upto == 1:
            return
        fused = decode and P <= 4 * E
        h = ops.grouped_gemm(xp, w.w13.blocks, E, I, True, counts, offsets, nt, out=hbuf, xsum=xs if decode else None,
                             workspace=gws[0], osum=hs if fused else None)
        if decode and not fused:
            ops.group_sums(h, offsets[E:], out=hs)
        if upto == 2:
            return
        y = ops.grouped_gemm(h, w.w2.blocks, E, H, False, counts, offsets, nt, out=yp,
                             xsum=hs if decode else None, workspace=gws[1])
        if upto == 3:
            return
        ops.moe_combine(y, pp, wts)

    prev = 0.0
    for upto in range(len(stages)):
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(2):
                layer(upto)
        torch.cuda.current_stream().wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            layer(upto)
        for _ in range(5):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 50 * 1e3
        print(f"{model} T={T} ntok={nt} ..{stages[upto]:14s} {us:8.1f} us  (+{us - prev:6.1f})", flush=True)
        prev = us


if __name__ == "__main__":
    a = sys.argv[1:]
    for i in range(0, len(a), 2):
        run(a[i], int(a[i + 1]))
