#!/usr/bin/env python
"""Every kernel of the library on small problems, once, for compute-sanitizer (memcheck, racecheck,
synccheck): routing (softmax / grouped top-k / fused route+permute), permutation (one CTA and
multi-CTA), gather (+ sums), group sums, the grouped GEMM in decode mode (16-token tiles with sums,
fused output sums, n-pair down, split-K) and prefill mode (16..128-token tiles), the fused-gather
GEMM, combine (activation and fp32), the EP localize and finalize paths, repack and dequant.

    compute-sanitizer --tool memcheck python tools/sanitize_all.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
from paper_2504_16214_b200.moe import ops  # noqa: E402
from paper_2504_16214_b200.moe.weights import random_packed  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    T, E, k, H, I = 37, 16, 4, 512, 256
    lg = torch.randn((T, E), device=dev, generator=g)
    ids, wts = ops.route_topk(lg, k, "softmax", True)
    ops.route_grouped_topk(lg, k, 4, 2, "sigmoid", True)
    ops.route_permute(lg, k, "softmax", True)
    P = T * k
    c, o, sp, pp = ops.moe_permute(ids, E)
    ws = torch.empty(max(ops.permute_ws_bytes(4096, E), 1), dtype=torch.uint8, device=dev)
    big = torch.randint(0, E, (1024, 4), dtype=torch.int32, device=dev, generator=g)
    ops.moe_permute(big, E, ws)
    x = (torch.randn((T, H), device=dev, generator=g) * 0.5).half()
    w13 = random_packed(E, 2 * I, H, True, torch.float16, g, dev)
    w2 = random_packed(E, H, I, False, torch.float16, g, dev)
    xp, xs = ops.moe_gather_sums(x, sp, k, P, o[E:])
    ops.moe_gather(x, sp, k, P, o[E:])
    hs = torch.empty(ops.sums_shape(P, I), dtype=torch.float32, device=dev)
    for nt in (16, 32, 64, 128):
        dec = nt == 16
        gu_ws = torch.zeros(max(ops.gemm_ws_bytes(P, H, E, I, True, nt), 1), dtype=torch.uint8, device=dev)
        h = ops.grouped_gemm(xp, w13.blocks, E, I, True, c, o, nt, xsum=xs if dec else None, workspace=gu_ws,
                             osum=hs if dec else None)
        if dec:
            ops.group_sums(h, o[E:], out=hs)
        dn_ws = torch.zeros(max(ops.gemm_ws_bytes(P, I, E, H, False, nt), 1), dtype=torch.uint8, device=dev)
        y = ops.grouped_gemm(h, w2.blocks, E, H, False, c, o, nt, xsum=hs if dec else None, workspace=dn_ws)
        ops.grouped_gemm_gather(x, sp, k, w13.blocks, E, I, True, c, o, nt, xsum=ops.group_sums(x) if dec else None,
                                rows=P)
        ops.moe_combine(y, pp, wts)
        ops.moe_combine(y, pp, wts, f32=True)
        torch.cuda.synchronize()
        print("ntok", nt, "ok", flush=True)
    # split-K (few tiles: one token, two experts)
    ids1 = torch.tensor([[1, 5]], dtype=torch.int32, device=dev)
    c1, o1, sp1, pp1 = ops.moe_permute(ids1, E)
    xp1, xs1 = ops.moe_gather_sums(x[:1], sp1, 2, 2, o1[E:])
    sk = torch.zeros(max(ops.gemm_ws_bytes(2, H, E, I, True, 16), 1), dtype=torch.uint8, device=dev)
    ops.grouped_gemm(xp1, w13.blocks, E, I, True, c1, o1, 16, xsum=xs1, workspace=sk)
    loc = ops.ep_localize(ids, 4, 8)
    ops.dequant(w2.blocks[: w2.blocks.numel() // E], 1, H, I, 1, torch.float16)
    torch.cuda.synchronize()
    print("all kernels ok", loc.shape, flush=True)


if __name__ == "__main__":
    main()
