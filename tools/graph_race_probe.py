#!/usr/bin/env python
"""Do back-to-back replays of the layer graph overlap? (They run ~12 % faster than replays separated
by any stream operation.) The layer is captured with its output written into its own
input buffer, x <- MoE(x), using only the library's (PDL-launched) kernels, so replay i+1 reads what
replay i wrote: if consecutive replays overlapped, the chained result would differ from the same
chain run eagerly with a synchronize after every layer."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2504_16214_b200.moe import ops, random_moe_weights  # noqa: E402

T, E, k, H, I = 64, 256, 8, 7168, 2048
P = T * k
dev = torch.device("cuda", 0)
dt = torch.bfloat16
w = random_moe_weights(E, H, I, dt, device=dev, seed=11)
g = torch.Generator(device=dev).manual_seed(5)
x0 = (torch.randn((T, H), device=dev, generator=g) * 0.5).to(dt)
lg = torch.randn((T, E), device=dev, generator=g)
x = x0.clone()
nt = ops.pick_ntok(P, E)
perm_ws = torch.empty(max(ops.permute_ws_bytes(P, E), 1), dtype=torch.uint8, device=dev)
xp = torch.empty((P, H), dtype=dt, device=dev)
xs = torch.empty(ops.sums_shape(P, H), dtype=torch.float32, device=dev)
hb = torch.empty((P, I), dtype=dt, device=dev)
hs = torch.empty(ops.sums_shape(P, I), dtype=torch.float32, device=dev)
yp = torch.empty((P, H), dtype=dt, device=dev)
gu_ws = torch.empty(max(ops.gemm_ws_bytes(P, H, E, I, True, nt), 1), dtype=torch.uint8, device=dev)
dn_ws = torch.empty(max(ops.gemm_ws_bytes(P, I, E, H, False, nt), 1), dtype=torch.uint8, device=dev)


def layer_into_x():
    ids, wts = ops.route_topk(lg, k, "softmax", True)
    counts, offsets, sp, pp = ops.moe_permute(ids, E, perm_ws)
    ops.moe_gather_sums(x, sp, k, P, offsets[E:], out=xp, sums=xs)
    ops.grouped_gemm(xp, w.w13.blocks, E, I, True, counts, offsets, nt, out=hb, xsum=xs, workspace=gu_ws, osum=hs)
    ops.grouped_gemm(hb, w.w2.blocks, E, H, False, counts, offsets, nt, out=yp, xsum=hs, workspace=dn_ws)
    ops.moe_combine(yp, pp, wts, out=x)


# eager chain, a synchronize after every layer
N = 4
x.copy_(x0)
ref = []
for _ in range(N):
    layer_into_x()
    torch.cuda.synchronize()
    ref.append(x.clone())
print("eager chain finite:", [bool(torch.isfinite(r.float()).all()) for r in ref],
      "| layer changes x:", not torch.equal(ref[0], ref[1]))

x.copy_(x0)
side = torch.cuda.Stream()
side.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(side):
    layer_into_x()
torch.cuda.current_stream().wait_stream(side)
gr = torch.cuda.CUDAGraph()
with torch.cuda.graph(gr):
    layer_into_x()
for trial in range(3):
    x.copy_(x0)
    torch.cuda.synchronize()
    for _ in range(N):
        gr.replay()  # back to back
    torch.cuda.synchronize()
    print(f"trial {trial}: {N} back-to-back replays == eager chain: {torch.equal(x, ref[-1])}")


def per_replay(gap: bool, n=40):
    x.copy_(x0)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        gr.replay()
        if gap:
            torch.cuda.current_stream().wait_event(a)  # a no-op dependency between replays
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


print(f"per replay: back to back {per_replay(False):.4f} ms, with an event wait between {per_replay(True):.4f} ms")
