#!/usr/bin/env python
"""Golden vectors from vLLM's own CUDA / Triton MoE kernels (run on a GPU box, vLLM 0.22 from the image):

* top-k routing: vllm._custom_ops.topk_softmax / topk_sigmoid (the `fused_topk` of vLLM's FusedMoE);
* the W4A16 MoE layer: vllm.model_executor.layers.fused_moe.fused_moe.fused_experts with
  int4_w4a16_moe_quant_config (vLLM's moe_wna16 Triton path for AWQ checkpoints: weights
  [E, N, K/2] uint8 low nibble = even k, zeros [E, N/2, K/G] uint8 low nibble = even n,
  scales [E, N, K/G]; converted here from the oracle's logical (q, z, s)).

Writes gpurun_out/golden_vllm.npz; committed as tests/golden/vllm_moe.npz (tests/test_oracle.py pins
the oracle to it on the CPU).

    gpurun -- python tools/make_golden_vllm.py
"""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT / "oracle"))
import moe_oracle as O  # noqa: E402


def main():
    import vllm._custom_ops as ops
    from vllm.model_executor.layers.fused_moe.config import int4_w4a16_moe_quant_config
    from vllm.model_executor.layers.fused_moe.fused_moe import fused_experts
    out = {}
    rng = np.random.default_rng(2024)
    # ---- routing
    cases = [(33, 8, 2, "softmax", True), (33, 8, 2, "softmax", False), (64, 256, 8, "softmax", True),
             (40, 128, 8, "softmax", False), (17, 64, 6, "sigmoid", True), (17, 64, 6, "sigmoid", False)]
    for ci, (T, E, k, sc, rn) in enumerate(cases):
        lg = rng.standard_normal((T, E)).astype(np.float32)
        lg[0, 3] = lg[0, 5]          # exact ties inside the top-k
        lg[1, :] = 0.25              # a row of all-equal logits
        g = torch.from_numpy(lg).cuda()
        w = torch.empty((T, k), dtype=torch.float32, device="cuda")
        ids = torch.empty((T, k), dtype=torch.int32, device="cuda")
        tei = torch.empty((T, k), dtype=torch.int32, device="cuda")
        (ops.topk_softmax if sc == "softmax" else ops.topk_sigmoid)(w, ids, tei, g, rn)
        torch.cuda.synchronize()
        out[f"route{ci}_logits"] = lg
        out[f"route{ci}_meta"] = np.array([T, E, k, int(sc == "softmax"), int(rn)])
        out[f"route{ci}_ids"] = ids.cpu().numpy()
        out[f"route{ci}_w"] = w.cpu().numpy()
    # ---- the layer
    for li, (T, E, k, H, I, dt) in enumerate([(33, 8, 2, 256, 256, "f16"), (21, 16, 4, 512, 256, "bf16")]):
        tdt = torch.float16 if dt == "f16" else torch.bfloat16
        q13, z13, s13 = O.synth_awq_expert_weights(rng, E, 2 * I, H, dt)
        q2, z2, s2 = O.synth_awq_expert_weights(rng, E, H, I, dt)
        x = O.round_act(rng.standard_normal((T, H)).astype(np.float32) * 0.5, dt)
        ids, wts = O.route_topk(rng.standard_normal((T, E)).astype(np.float32), k, "softmax", True)

        def wna16(q, z, s):
            qw = (q[:, :, 0::2] | (q[:, :, 1::2] << 4)).astype(np.uint8)                      # [E, N, K/2]
            qz = (z[:, 0::2, :] | (z[:, 1::2, :] << 4)).astype(np.uint8)                      # [E, N/2, K/G]
            return (torch.from_numpy(qw).cuda(), torch.from_numpy(s).cuda().to(tdt), torch.from_numpy(qz).cuda())
        w1, s1, zp1 = wna16(q13, z13, s13)
        w2, s2_, zp2 = wna16(q2, z2, s2)
        qc = int4_w4a16_moe_quant_config(w1_scale=s1, w2_scale=s2_, w1_zp=zp1, w2_zp=zp2, block_shape=[0, 128])
        xd = torch.from_numpy(x).cuda().to(tdt)
        y = fused_experts(xd, w1, w2, torch.from_numpy(wts).cuda(), torch.from_numpy(ids).cuda(), quant_config=qc)
        torch.cuda.synchronize()
        for name, v in (("q13", q13), ("z13", z13), ("s13", s13), ("q2", q2), ("z2", z2), ("s2", s2), ("x", x),
                        ("ids", ids), ("w", wts)):
            out[f"layer{li}_{name}"] = v
        out[f"layer{li}_meta"] = np.array([T, E, k, H, I, int(dt == "f16")])
        out[f"layer{li}_y"] = y.float().cpu().numpy()
    Path(ROOT / "gpurun_out").mkdir(exist_ok=True)
    np.savez_compressed(ROOT / "gpurun_out" / "golden_vllm.npz", **out)
    print("wrote", len(out), "arrays; vllm", __import__("vllm").__version__)


if __name__ == "__main__":
    main()
