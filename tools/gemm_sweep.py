#!/usr/bin/env python
"""Per-kernel CUDA-event times of the DS-R1 W4A16 MoE layer across token counts and token-tile
sizes (GPU). Prints one JSON line per (T, ntok) with each kernel's mean ms and the gate/up and down
GEMMs' achieved GB/s (algorithmic bytes).

    python tools/gemm_sweep.py [--tokens 1,16,64] [--ntok 0,16,32,64,128] [--reps 10]
"""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
E_DS = K_DS = H_DS = I_DS = 0  # layer shape, set from --model


def main():
    import torch
    from bench import w_bytes
    from paper_2504_16214_b200.moe import moe_w4a16, random_moe_weights, select_experts
    from paper_2504_16214_b200.moe.layer import KernelTimer
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", default="1,4,16,64,256,1024,4096,8192")
    ap.add_argument("--ntok", default="0")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--dtype", default="f16")
    ap.add_argument("--model", default="ds", choices=["ds", "mixtral", "qwen3"])
    a = ap.parse_args()
    global E_DS, K_DS, H_DS, I_DS
    E_DS, K_DS, H_DS, I_DS = {"ds": (256, 8, 7168, 2048), "mixtral": (8, 2, 4096, 14336),
                              "qwen3": (128, 8, 2048, 768)}[a.model]
    dev = torch.device("cuda", 0)
    tdt = torch.float16 if a.dtype == "f16" else torch.bfloat16
    w = random_moe_weights(E_DS, H_DS, I_DS, tdt, device=dev, seed=7)
    g = torch.Generator().manual_seed(0)
    for T in map(int, a.tokens.split(",")):
        x = (torch.randn((T, H_DS), generator=g) * 0.5).to(tdt).to(dev)
        lg = torch.randn((T, E_DS), generator=g).to(dev)
        wts, ids = select_experts(lg, K_DS, "softmax", True)
        counts = torch.bincount(ids.flatten().long(), minlength=E_DS)
        et = int((counts > 0).sum())
        for nt in map(int, a.ntok.split(",")):
            try:
                for _ in range(3):
                    moe_w4a16(x, w, wts, ids, ntok=nt)
                torch.cuda.synchronize()
                tm = KernelTimer()
                for _ in range(a.reps):
                    moe_w4a16(x, w, wts, ids, ntok=nt, timer=tm)
                torch.cuda.synchronize()
            except Exception as e:  # noqa: BLE001
                print(json.dumps({"T": T, "ntok": nt, "error": repr(e)}))
                continue
            ms = {k: round(tm.mean_ms(k), 4) for k in tm.events}
            P = T * K_DS
            gu_b = et * w_bytes(2 * I_DS, H_DS) + P * (H_DS + I_DS) * 2
            dn_b = et * w_bytes(H_DS, I_DS) + P * (I_DS + H_DS) * 2
            print(json.dumps({"T": T, "ntok": nt, "experts": et, "max_count": int(counts.max()), "ms": ms,
                              "total_ms": round(sum(ms.values()), 4),
                              "gate_up_GBs": round(gu_b / ms["gemm_gate_up"] / 1e6, 1),
                              "down_GBs": round(dn_b / ms["gemm_down"] / 1e6, 1),
                              "gate_up_TFs": round(4 * P * H_DS * I_DS / ms["gemm_gate_up"] / 1e9, 1),
                              "down_TFs": round(2 * P * H_DS * I_DS / ms["gemm_down"] / 1e9, 1)}), flush=True)


if __name__ == "__main__":
    main()
