#!/usr/bin/env python
"""Run the grouped GEMM variants (gate/up and k-pair down, offset and prefill modes) on small
random problems, optionally many times, to flush out hangs/races (use under compute-sanitizer or
with a short `timeout`). Prints one line per variant."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402
from paper_2504_16214_b200.moe import ops  # noqa: E402
from paper_2504_16214_b200.moe.weights import random_packed  # noqa: E402


def main(reps=1, E=6, H=512, I=384):
    dev = torch.device("cuda", 0)
    g = torch.Generator(device="cpu").manual_seed(0)
    counts = torch.tensor([5, 0, 17, 1, 40, 130][:E], dtype=torch.int32)
    off = torch.zeros(E + 1, dtype=torch.int32)
    off[1:] = torch.cumsum(counts, 0)
    rows = int(off[-1])
    counts, off = counts.to(dev), off.to(dev)
    gd = torch.Generator(device=dev).manual_seed(1)
    w13 = random_packed(E, 2 * I, H, True, torch.float16, gd, dev)
    w2 = random_packed(E, H, I, False, torch.float16, gd, dev)
    x = (torch.randn((rows, H), generator=g) * 0.5).half().to(dev)
    h = (torch.randn((rows, I), generator=g) * 0.5).half().to(dev)
    for ntok in (16, 32, 64, 128):
        for name, fn in (("gate_up", lambda: ops.grouped_gemm(x, w13.blocks, E, I, True, counts, off, ntok)),
                         ("down", lambda: ops.grouped_gemm(h, w2.blocks, E, H, False, counts, off, ntok))):
            t0 = time.time()
            for _ in range(reps):
                fn()
            torch.cuda.synchronize()
            print(f"{name} ntok={ntok} reps={reps} ok {time.time() - t0:.2f}s", flush=True)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 1)
