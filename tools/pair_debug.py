#!/usr/bin/env python
"""Run one grouped GEMM and save its output (compare a W4A16_PREFILL_PAIR=1 run with a default run):
    python tools/pair_debug.py save OUT.npy --counts 128 --n 256 --k 128 --gated 0 --ntok 128
    python tools/pair_debug.py diff A.npy B.npy --ntok 128"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("cmd")
ap.add_argument("files", nargs="+")
ap.add_argument("--counts", default="128")
ap.add_argument("--n", type=int, default=256)
ap.add_argument("--k", type=int, default=128)
ap.add_argument("--gated", type=int, default=0)
ap.add_argument("--ntok", type=int, default=128)
a = ap.parse_args()
if a.cmd == "save":
    import torch
    from paper_2504_16214_b200.moe import ops
    from paper_2504_16214_b200.moe.weights import random_packed
    dev = torch.device("cuda", 0)
    counts = [int(c) for c in a.counts.split(",")]
    E = len(counts)
    g = torch.Generator(device=dev).manual_seed(3)
    w = random_packed(E, 2 * a.n if a.gated else a.n, a.k, bool(a.gated), torch.float16, g, dev)
    rows = sum(counts)
    x = (torch.randn((rows, a.k), generator=g, device=dev) * 0.5).half()
    cnt = torch.tensor(counts, dtype=torch.int32, device=dev)
    off = torch.zeros(E + 1, dtype=torch.int32, device=dev)
    off[1:] = torch.cumsum(cnt, 0)
    y = ops.grouped_gemm(x, w.blocks, E, a.n, bool(a.gated), cnt, off, a.ntok)
    torch.cuda.synchronize()
    np.save(a.files[0], y.float().cpu().numpy())
else:
    A, B = np.load(a.files[0]), np.load(a.files[1])
    bad = ~np.isclose(A, B, rtol=1e-2, atol=1e-2)
    print("shape", A.shape, "bad", int(bad.sum()), "of", bad.size)
    if bad.any():
        r, c = np.nonzero(bad)
        print("bad rows", np.unique(r)[:40], "... n", len(np.unique(r)))
        print("bad col tiles (128)", np.unique(c // 128), "bad cols mod 128 sample", np.unique(c % 128)[:40])
        for rr in np.unique(r)[:3]:
            cc = np.nonzero(bad[rr])[0][:8]
            print(" row", rr, "cols", cc, "A", A[rr, cc], "B", B[rr, cc])
