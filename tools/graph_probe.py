#!/usr/bin/env python
"""Per-replay time of the DS-R1 T=64 layer as a CUDA graph, back to back and with an event record
between replays, for graphs with/without a tiny plain (non-PDL) kernel before / after the layer
(GPU). Diagnoses the ~0.15 ms a stream operation between replays of the plain layer graph costs."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
from paper_2504_16214_b200.moe import _lib, fused_moe_w4a16, random_moe_weights  # noqa: E402

T, E, K, H, I = 64, 256, 8, 7168, 2048
dev = torch.device("cuda", 0)
w = random_moe_weights(E, H, I, torch.float16, device=dev, seed=7)
x = (torch.randn((T, H)) * 0.5).half().cuda()
lg = torch.randn((T, E)).cuda()
buf = torch.zeros(4096, dtype=torch.int64, device=dev)
side = torch.cuda.Stream()
side.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(side):
    for _ in range(2):
        fused_moe_w4a16(x, lg, w, K, "softmax", True)
torch.cuda.current_stream().wait_stream(side)


def stamp():
    _lib.call("w4a16_debug_stamp", buf.data_ptr(), torch.cuda.current_stream().cuda_stream)


def capture(pre, post):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        if pre:
            stamp()
        fused_moe_w4a16(x, lg, w, K, "softmax", True)
        if post:
            stamp()
    return g


ev = torch.cuda.Event()
for pre, post in ((False, False), (True, False), (False, True), (True, True)):
    g = capture(pre, post)
    res = []
    for between in (False, True):
        for _ in range(5):
            g.replay()
        torch.cuda.synchronize()
        buf.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(40):
            g.replay()
            if between:
                ev.record()
        e1.record()
        torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) / 40)
    print(f"graph [{'stamp, ' if pre else ''}layer{', stamp' if post else ''}]: back to back {res[0]:.4f} ms, "
          f"event between {res[1]:.4f} ms")

# globaltimer sanity: stamped duration vs CUDA-event duration of the same replays
g = capture(True, True)
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
buf.zero_()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    g.replay()
e1.record()
torch.cuda.synchronize()
n = int(buf[0].item())
ts = buf[1:1 + n].cpu().double()
print(f"20 replays: CUDA events {e0.elapsed_time(e1):.3f} ms, globaltimer first->last stamp {(ts.max() - ts.min()).item() / 1e6:.3f} ms")

# where does a replay's time go? stamps around every kernel of the layer (inside the graph)


class StampTimer:
    names: list = []

    def span(self, name):
        class _S:
            def __enter__(s):
                StampTimer.names.append(name)
                stamp()

            def __exit__(s, *exc):
                stamp()
        return _S()


st_ = StampTimer()
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(side):
    fused_moe_w4a16(x, lg, w, K, "softmax", True, timer=StampTimer())
torch.cuda.synchronize()
StampTimer.names = []
with torch.cuda.graph(g):
    fused_moe_w4a16(x, lg, w, K, "softmax", True, timer=st_)
names = list(StampTimer.names)
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
buf.zero_()
for _ in range(10):
    g.replay()
torch.cuda.synchronize()
n = int(buf[0].item())
ts = buf[1:1 + n].cpu().double().view(10, -1)
ts = ts.sort(dim=1).values
d = (ts[:, 1:] - ts[:, :-1]).median(dim=0).values / 1e3
parts = []
for i, nm in enumerate(names):
    parts.append(f"{nm} {d[2 * i].item():.1f}")
    if 2 * i + 1 < d.numel():
        parts.append(f"gap {d[2 * i + 1].item():.1f}")
print("per-kernel us (stamped graph):", ", ".join(parts), f"| replay {((ts[:, -1] - ts[:, 0]).median() / 1e3).item():.1f} us")
