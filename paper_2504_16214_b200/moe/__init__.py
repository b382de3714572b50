"""W4A16 mixture-of-experts operator on B200 (sm_100a CUDA kernels behind a C ABI)."""
from .layer import FusedMoEGraph, FusedMoEPipeline, fused_moe_w4a16, moe_w4a16, select_experts, w4a16_linear
from .checkpoint import load_awq_moe, load_packed, save_packed
from .vllm_method import W4A16MoEMethod
from .weights import MoEWeights, PackedW4, pack_awq, pack_moe_awq, random_moe_weights

__all__ = [
    "FusedMoEGraph",
    "FusedMoEPipeline",
    "MoEWeights",
    "PackedW4",
    "W4A16MoEMethod",
    "fused_moe_w4a16",
    "load_awq_moe",
    "load_packed",
    "moe_w4a16",
    "pack_awq",
    "pack_moe_awq",
    "random_moe_weights",
    "save_packed",
    "select_experts",
    "w4a16_linear",
]
