#!/usr/bin/env python
"""Where does the end-to-end step time go? Times the DS-R1 T=64 layer through FusedMoEPipeline with
and without the host copies (GPU)."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402
from paper_2504_16214_b200.moe import FusedMoEPipeline, random_moe_weights  # noqa: E402

T, E, K, H, I = 64, 256, 8, 7168, 2048
dev = torch.device("cuda", 0)
w = random_moe_weights(E, H, I, torch.float16, device=dev, seed=7)
x_h = (torch.randn((T, H)) * 0.5).half().pin_memory()
lg_h = torch.randn((T, E)).pin_memory()
y_h = torch.empty((T, H), dtype=torch.float16).pin_memory()
pipe = FusedMoEPipeline(w, T, K, "softmax", True, torch.float16, dev, x=x_h.cuda(), router_logits=lg_h.cuda())
g = pipe.slots[0]
steps = 50


def timed(fn, label):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"{label:40s} {e0.elapsed_time(e1) / steps:.4f} ms/step (host enqueue {1e3 * (t1 - t0) / steps:.4f} ms/step)")


def pipe_steps():
    pipe.start()
    pipe(x_h, lg_h, y_h)
    pipe.finish()


timed(lambda: g.graph.replay(), "graph replay only")
timed(pipe_steps, "pipeline (H2D + layer + D2H)")
xd, ld = x_h.cuda(), lg_h.cuda()
timed(lambda: (g.x.copy_(x_h, non_blocking=True), g.logits.copy_(lg_h, non_blocking=True), g.graph.replay()),
      "serial H2D + layer")
timed(lambda: (g.graph.replay(), y_h.copy_(g.y, non_blocking=True)), "serial layer + D2H")
timed(lambda: (g.x.copy_(x_h, non_blocking=True), g.logits.copy_(lg_h, non_blocking=True), g.graph.replay(),
               y_h.copy_(g.y, non_blocking=True)), "serial H2D + layer + D2H")
scratch = torch.zeros(16, device=dev)
timed(lambda: (scratch.add_(1), g.graph.replay()), "tiny torch kernel + layer")
xd2 = torch.empty_like(g.x)
timed(lambda: (g.x.copy_(xd2, non_blocking=True), g.graph.replay()), "D2D copy + layer")
# H2D + layer + D2H captured in ONE graph (fixed pinned host buffers)
from paper_2504_16214_b200.moe import fused_moe_w4a16  # noqa: E402
g2 = torch.cuda.CUDAGraph()
s2 = torch.cuda.Stream()
s2.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s2):
    for _ in range(2):
        g.x.copy_(x_h, non_blocking=True)
        yy = fused_moe_w4a16(g.x, g.logits, w, K, "softmax", True)
torch.cuda.current_stream().wait_stream(s2)
with torch.cuda.graph(g2):
    g.x.copy_(x_h, non_blocking=True)
    g.logits.copy_(lg_h, non_blocking=True)
    yy = fused_moe_w4a16(g.x, g.logits, w, K, "softmax", True)
    y_h.copy_(yy, non_blocking=True)
timed(lambda: g2.replay(), "one graph: H2D + layer + D2H")
timed(lambda: (g.graph.replay(), g.graph.replay(), scratch.add_(1)), "2 replays + tiny kernel (per 2)")
timed(lambda: g.x.copy_(x_h, non_blocking=True), "H2D x only")
timed(lambda: y_h.copy_(g.y, non_blocking=True), "D2H y only")
