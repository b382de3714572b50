#!/usr/bin/env python
"""Per-stage timeline of CTA 0 of one grouped-GEMM launch (w4a16_debug_trace): prints the mean
interval between the roles' sync points in steady state. --which gate_up|down."""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2504_16214_b200.moe import _lib, ops  # noqa: E402
from paper_2504_16214_b200.moe.weights import random_packed  # noqa: E402

EV = ["prod_empty_ok", "dq_full_ok", "dq_aempty_ok", "dq_afull_arrive", "mma_ready", "mma_issued",
      "epi_full_ok", "epi_accfull_ok", "epi_done", "epi_tile_start"]

ap = argparse.ArgumentParser()
ap.add_argument("--which", default="gate_up")
ap.add_argument("--experts", type=int, default=224)
ap.add_argument("--per-expert", type=int, default=2)
ap.add_argument("--ntok", type=int, default=16)
ap.add_argument("--cta", type=int, default=0, help="CTA whose timeline is recorded")
ap.add_argument("--nk", default="", help="N,K override (e.g. 14336,4096 for the Llama-3-8B linear)")
ap.add_argument("--dump", action="store_true", help="every stage's MMA-ready / epilogue-done time")
ap.add_argument("--xscale", type=float, default=0.5, help="0 = all-zero activations (data-dependent power probe)")
a = ap.parse_args()
H, I = 7168, 2048
dev = torch.device("cuda", 0)
E = a.experts
gd = torch.Generator(device=dev).manual_seed(1)
gated = a.which == "gate_up"
N, K = (2 * I, H) if gated else (H, I)
if a.nk:
    N, K = (int(v) for v in a.nk.split(","))
    N = 2 * N if gated else N
w = random_packed(E, N, K, gated, torch.float16, gd, dev)
counts = torch.full((E,), a.per_expert, dtype=torch.int32, device=dev)
off = torch.zeros(E + 1, dtype=torch.int32, device=dev)
off[1:] = torch.cumsum(counts, 0)
x = (torch.randn((E * a.per_expert, K), device=dev) * a.xscale).half()
nout = N // 2 if gated else N
xs = ops.group_sums(x) if a.ntok <= 32 else None
rows = E * a.per_expert
ws = torch.zeros(max(ops.gemm_ws_bytes(rows, K, E, nout, gated, a.ntok), 1), dtype=torch.uint8, device=dev)
for _ in range(2):
    ops.grouped_gemm(x, w.blocks, E, nout, gated, counts, off, a.ntok, xsum=xs, workspace=ws)
buf = torch.full((30, 4096), -1, dtype=torch.int64, device=dev)
_lib.call("w4a16_debug_trace_cta", a.cta)
_lib.call("w4a16_debug_trace", buf.data_ptr())
torch.cuda.synchronize()
ops.grouped_gemm(x, w.blocks, E, nout, gated, counts, off, a.ntok, xsum=xs, workspace=ws)
torch.cuda.synchronize()
_lib.call("w4a16_debug_trace", None)
t = buf.cpu().numpy()
n = int(max((t[4] >= 0).sum(), (t[1] >= 0).sum()))  # the peer CTA of a pair records no MMA events
t0 = t[t >= 0].min()
t = np.where(t >= 0, t - t0, -1)
lo, hi = n // 4, 3 * n // 4
s = slice(lo, hi)
print(f"{a.which}: stages traced {n}, steady window [{lo},{hi}); CTA span (first to last event) {t.max()} cyc")
per = np.diff(t[4][s] if (t[4] >= 0).sum() else t[1][s]).mean()
print(f"  stage period (mma_ready diffs)          {per:8.1f} cyc")
def m(x):
    return float(np.mean(x))
print(f"  dequant: full_ok -> aempty_ok            {m(t[2][s] - t[1][s]):8.1f}")
print(f"  dequant: aempty_ok -> afull arrive       {m(t[3][s] - t[2][s]):8.1f}")
print(f"  mma: afull arrive -> mma_ready           {m(t[4][s] - t[3][s]):8.1f}")
print(f"  mma: ready -> issued                     {m(t[5][s] - t[4][s]):8.1f}")
print(f"  epi: mma_issued -> accfull_ok            {m(t[7][s] - t[5][s]):8.1f}")
print(f"  epi: accfull_ok -> done                  {m(t[8][s] - t[7][s]):8.1f}")
print(f"  epi: full_ok -> accfull_ok               {m(t[7][s] - t[6][s]):8.1f}")
print(f"  producer: empty_ok(gs) - mma_ready(gs)   {m(t[0][s] - t[4][s]):8.1f}")
print(f"  dq aempty_ok(gs) - mma_issued(gs-3)      {m(t[2][lo + 3:hi] - t[5][lo:hi - 3]):8.1f}")
print(f"  mma_ready(gs) - epi_done(gs-2)           {m(t[4][lo + 2:hi] - t[8][lo:hi - 2]):8.1f}")
print(f"  full_ok(dq) - prod_empty_ok (load lat)   {m(t[1][s] - t[0][s]):8.1f}")
if (t[16] >= 0).sum() > 8:  # per-quad afull arrival (rows 16..19), relative to quad 0
    q = [t[16 + i][s] for i in range(4)]
    print("  afull arrival per quad rel. to quad 0:", [round(m(q[i] - q[0]), 1) for i in range(4)],
          f" MMA ready - last arrival {m(t[4][s] - np.max(np.stack(q), axis=0)):.1f}")
if (t[20] >= 0).sum() > 8:
    print(f"  MMA warp: issued -> commits accepted {m(t[20][s] - t[5][s]):8.1f}, -> reconverged {m(t[21][s] - t[5][s]):8.1f}, "
          f"reconverged -> next ready {m(t[4][lo + 1:hi + 1] - t[21][s]):8.1f}")
if a.ntok > 32:  # prefill: per-tile epilogue (events 6-8 indexed by tile)
    nt_ = int((t[7] >= 0).sum())
    if nt_ > 2:
        print(f"  prefill tiles {nt_}: epilogue accfull_ok -> done   {m(t[8][:nt_] - t[7][:nt_]):8.1f}")
        print(f"  MMA tile start (accempty ok) - prev accfull_ok  {m(t[6][1:nt_] - t[7][:nt_ - 1]):8.1f}")
        e = t[14][: nt_ * 32].reshape(nt_, 32)[1:-1]
        print("  epilogue per 16-token chunk: [ld-wait done, stores done] rel. to accfull_ok, mean over tiles:")
        print("   ", np.round((e - t[7][1:nt_ - 1, None]).mean(0)).astype(int).tolist())
        print(f"  tile period                                     {m(np.diff(t[7][:nt_])):8.1f}")
if (t[15] >= 0).sum() > 8:  # MMA completion per stage (non-offset, trace build)
    c = t[15][s]
    print(f"  MMA complete period                              {np.diff(c).mean():8.1f}")
    print(f"  MMA complete(gs) - issued(gs)                    {m(c - t[5][s]):8.1f}")
    busy = np.minimum(np.diff(c), c[1:] - t[5][lo + 1:hi])
    print(f"  stage exec est. (complete - max(prev complete, issued)) {m(busy):8.1f}")
    print(f"  MMA issued(gs) - complete(gs-1) (<0: queued behind)      {m(t[5][lo + 1:hi] - c[:-1]):8.1f}")
ts = t[9][t[9] >= 0]
print(f"  tiles traced {len(ts)}")
print("  first 12 stages (cycles rel.):")
for i in range(lo, lo + 12):
    print("   ", i, " ".join(f"{EV[e][:10]}={t[e][i]}" for e in (0, 1, 2, 3, 4, 5, 7, 8)))

if a.dump:
    print("  stage: prod_empty_ok dq_full_ok mma_ready mma_issued epi_accfull epi_done (cycles from the first event)")
    r = buf.cpu().numpy()[:10]
    z = r[r >= 0].min()
    r = np.where(r >= 0, r - z, -1)
    for i in range(n):
        print(f"  S{i:3d} {r[0][i]:8d} {r[1][i]:8d} {r[4][i]:8d} {r[5][i]:8d} {r[7][i]:8d} {r[8][i]:8d}")
    print("  epilogue tile starts:", r[9][r[9] >= 0].tolist(), " last epilogue done:", int(r[8].max()))
    w26 = buf.cpu().numpy()[26][:16]
    print("  warp arrivals at the exit barrier:", [int(v - z) if v >= 0 else -1 for v in w26])

if a.dump:
    g = buf.cpu().numpy()[28:30, :148]
    ok = g[0] > 0
    if ok.any():
        t0 = g[0][ok].min()
        ent, ex = (g[0][ok] - t0) / 1e3, (g[1][ok] - t0) / 1e3
        order = np.argsort(-ex)
        print(f"  CTA entry (us): min {ent.min():.2f} max {ent.max():.2f}; exit: min {ex.min():.2f} median "
              f"{np.median(ex):.2f} max {ex.max():.2f}; latest CTAs: " +
              ", ".join(f"{int(np.nonzero(ok)[0][j])}@{ex[j]:.2f}" for j in order[:6]))
