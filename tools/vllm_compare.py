#!/usr/bin/env python
"""vLLM 0.22's own W4A16 MoE paths vs this repository's layer, same DeepSeek-R1 shapes and routing,
graphed, one B200: (1) fused_marlin_moe on awq_marlin_moe_repack'ed weights -- what vLLM's
AWQMarlinMoEMethod runs for AWQ MoE checkpoints on NVIDIA GPUs; (2) fused_experts with
int4_w4a16_moe_quant_config (the moe_wna16 Triton kernels, default config: vLLM ships no tuned
B200 table for it). Prints ms per call for each token count.

    python tools/vllm_compare.py [1,64,256,8192]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

E, K, H, I = 256, 8, 7168, 2048


def timed(fn, reps=10):
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for _ in range(2):
            fn()
    torch.cuda.current_stream().wait_stream(side)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    from vllm.model_executor.layers.fused_moe.config import int4_w4a16_moe_quant_config
    from vllm.model_executor.layers.fused_moe.fused_moe import fused_experts
    from paper_2504_16214_b200.moe import moe_w4a16, random_moe_weights, select_experts
    dev = torch.device("cuda", 0)
    Ts = [int(t) for t in (sys.argv[1] if len(sys.argv) > 1 else "1,64,256,2048,8192").split(",")]
    ours = random_moe_weights(E, H, I, torch.float16, device=dev, seed=9)
    g = torch.Generator(device=dev).manual_seed(0)
    # vLLM moe_wna16 tensors of the same sizes (random codes: throughput depends on shapes, not values)
    w1 = torch.randint(0, 256, (E, 2 * I, H // 2), dtype=torch.uint8, device=dev, generator=g)
    w2 = torch.randint(0, 256, (E, H, I // 2), dtype=torch.uint8, device=dev, generator=g)
    s1 = (torch.rand((E, 2 * I, H // 128), device=dev, generator=g) * 0.01).half()
    s2 = (torch.rand((E, H, I // 128), device=dev, generator=g) * 0.01).half()
    z1 = torch.randint(0, 256, (E, I, H // 128), dtype=torch.uint8, device=dev, generator=g)
    z2 = torch.randint(0, 256, (E, H // 2, I // 128), dtype=torch.uint8, device=dev, generator=g)
    qc = int4_w4a16_moe_quant_config(w1_scale=s1, w2_scale=s2, w1_zp=z1, w2_zp=z2, block_shape=[0, 128])
    del w1, w2  # (kept out of the Marlin arm's memory)
    w1 = w2 = None
    from vllm import _custom_ops as vops
    from vllm.model_executor.layers.fused_moe.experts.marlin_moe import fused_marlin_moe
    from vllm.model_executor.layers.quantization.utils.marlin_utils import (marlin_make_workspace_new,
                                                                            marlin_moe_permute_scales,
                                                                            moe_awq_to_marlin_zero_points)
    from vllm.scalar_type import scalar_types
    ri = lambda *shape: torch.randint(-2**31, 2**31 - 1, shape, dtype=torch.int32, device=dev, generator=g)  # noqa
    sort = torch.empty((E, 0), dtype=torch.int32, device=dev)
    mw13 = vops.awq_marlin_moe_repack(ri(E, H, 2 * I // 8), sort, size_k=H, size_n=2 * I, num_bits=4)
    mw2 = vops.awq_marlin_moe_repack(ri(E, I, H // 8), sort, size_k=I, size_n=H, num_bits=4)
    ms13 = marlin_moe_permute_scales((torch.rand((E, H // 128, 2 * I), device=dev, generator=g) * 0.01).half(),
                                     size_k=I, size_n=2 * I, group_size=128)
    ms2 = marlin_moe_permute_scales((torch.rand((E, I // 128, H), device=dev, generator=g) * 0.01).half(),
                                    size_k=I, size_n=H, group_size=128)
    mz13 = moe_awq_to_marlin_zero_points(ri(E, H // 128, 2 * I // 8), size_k=H // 128, size_n=2 * I, num_bits=4)
    mz2 = moe_awq_to_marlin_zero_points(ri(E, I // 128, H // 8), size_k=I // 128, size_n=H, num_bits=4)
    mws = marlin_make_workspace_new(dev, 4)
    for T in Ts:
        x = (torch.randn((T, H), device=dev, generator=g) * 0.5).half()
        lg = torch.randn((T, E), device=dev, generator=g)
        wts, ids = select_experts(lg, K, "softmax", True)
        t_m = timed(lambda: fused_marlin_moe(x, mw13, mw2, None, None, ms13, ms2, wts, ids,
                                             quant_type_id=scalar_types.uint4.id, w1_zeros=mz13, w2_zeros=mz2,
                                             workspace=mws))
        t_o = timed(lambda: moe_w4a16(x, ours, wts, ids))
        print(f"T={T}: vLLM fused_marlin_moe {t_m:.3f} ms, this repo {t_o:.3f} ms, speed-up {t_m / t_o:.2f}x",
              flush=True)


if __name__ == "__main__":
    main()
