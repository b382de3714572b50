#!/usr/bin/env python
"""Which part of the layer makes back-to-back replays of one CUDA graph faster than replays
separated by a stream operation? Graphs of growing prefixes of the DS-R1 T=64 decode layer, each
timed back to back and with a wait on a completed event between replays (GPU)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
from paper_2504_16214_b200.moe import ops, random_moe_weights, select_experts  # noqa: E402

T, E, K, H, I = 64, 256, 8, 7168, 2048
dev = torch.device("cuda", 0)
w = random_moe_weights(E, H, I, torch.float16, device=dev, seed=7)
x = (torch.randn((T, H)) * 0.5).half().cuda()
lg = torch.randn((T, E)).cuda()
P = T * K
perm_ws = torch.empty(max(ops.permute_ws_bytes(P, E), 1), dtype=torch.uint8, device=dev)
xp = torch.empty((P, H), dtype=torch.float16, device=dev)
xs = torch.empty(ops.sums_shape(P, H), dtype=torch.float32, device=dev)
hbuf = torch.empty((P, I), dtype=torch.float16, device=dev)
hs = torch.empty(ops.sums_shape(P, I), dtype=torch.float32, device=dev)
yp = torch.empty((P, H), dtype=torch.float16, device=dev)
STAGES = ["route", "permute", "gather", "gate_up", "sums_h", "down", "combine"]


def layer(upto):
    wts, ids = select_experts(lg, K, "softmax", True)
    if upto == 0:
        return
    counts, offsets, sp, pp = ops.moe_permute(ids, E, perm_ws)
    if upto == 1:
        return
    ops.moe_gather_sums(x, sp, K, P, offsets[E:], out=xp, sums=xs)
    if upto == 2:
        return
    h = ops.grouped_gemm(xp, w.w13.blocks, E, I, True, counts, offsets, 16, out=hbuf, xsum=xs)
    if upto == 3:
        return
    ops.group_sums(h, offsets[E:], out=hs)
    if upto == 4:
        return
    y = ops.grouped_gemm(h, w.w2.blocks, E, H, False, counts, offsets, 16, out=yp, xsum=hs)
    if upto == 5:
        return
    ops.moe_combine(y, pp, wts)


done = torch.cuda.Event()
done.record()
side = torch.cuda.Stream()
for upto in range(len(STAGES)):
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for _ in range(2):
            layer(upto)
    torch.cuda.current_stream().wait_stream(side)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        layer(upto)
    res = []
    for between in (False, True):
        for _ in range(5):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(40):
            g.replay()
            if between:
                torch.cuda.current_stream().wait_event(done)
        e1.record()
        torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) / 40 * 1e3)
    print(f"graph route..{STAGES[upto]:8s}: back to back {res[0]:7.1f} us, wait between {res[1]:7.1f} us, "
          f"diff {res[1] - res[0]:6.1f}")

# stamps around the two GEMMs only (mid-graph), full layer, back to back vs wait between
from paper_2504_16214_b200.moe import _lib  # noqa: E402
buf = torch.zeros(8192, dtype=torch.int64, device=dev)


def stamp():
    _lib.call("w4a16_debug_stamp", buf.data_ptr(), torch.cuda.current_stream().cuda_stream)


def layer_stamped():
    wts, ids = select_experts(lg, K, "softmax", True)
    counts, offsets, sp, pp = ops.moe_permute(ids, E, perm_ws)
    ops.moe_gather_sums(x, sp, K, P, offsets[E:], out=xp, sums=xs)
    stamp()
    h = ops.grouped_gemm(xp, w.w13.blocks, E, I, True, counts, offsets, 16, out=hbuf, xsum=xs)
    stamp()
    ops.group_sums(h, offsets[E:], out=hs)
    stamp()
    y = ops.grouped_gemm(h, w.w2.blocks, E, H, False, counts, offsets, 16, out=yp, xsum=hs)
    stamp()
    ops.moe_combine(y, pp, wts)


side.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(side):
    for _ in range(2):
        layer_stamped()
torch.cuda.current_stream().wait_stream(side)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    layer_stamped()
for between in (False, True):
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    buf.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(30):
        g.replay()
        if between:
            torch.cuda.current_stream().wait_event(done)
    e1.record()
    torch.cuda.synchronize()
    n = int(buf[0].item())
    t = buf[1:1 + n].cpu().double().view(30, 4) / 1e3
    gu = (t[:, 1] - t[:, 0]).median().item()
    dn = (t[:, 3] - t[:, 2]).median().item()
    rest = (t[1:, 0] - t[:-1, 3]).median().item()
    print(f"stamped full layer, {'wait between' if between else 'back to back'}: {e0.elapsed_time(e1) / 30 * 1e3:.1f} us/replay; "
          f"gate/up {gu:.1f} us, down {dn:.1f} us, down end -> next gate/up start {rest:.1f} us")
