"""A vLLM-style FusedMoE quantisation method for this W4A16 path.

``W4A16MoEMethod`` has the shape of vLLM's ``AWQMarlinMoEMethod``
(vllm/model_executor/layers/quantization/awq_marlin.py:510-700): ``create_weights`` registers the same
AWQ parameters on the layer module (``w13_qweight [E, H, 2I/8] int32``, ``w13_scales [E, H/G, 2I]``,
``w13_qzeros [E, H/G, 2I/8] int32``, ``w2_*`` with K = I), the checkpoint loader fills them,
``process_weights_after_loading`` repacks them ONCE into this library's block format (replacing
the Marlin repack) and releases the AWQ copies, and ``apply`` runs the layer. It is duck-typed --
vLLM is not imported -- so it plugs into a FusedMoE layer object or any ``torch.nn.Module`` that
holds the parameters (the test drives it on a plain module).
"""
from __future__ import annotations

import torch
from torch.nn import Parameter

from .layer import fused_moe_w4a16, moe_w4a16
from .weights import pack_moe_awq

_AWQ_PARAMS = ("w13_qweight", "w13_scales", "w13_qzeros", "w2_qweight", "w2_scales", "w2_qzeros")


class W4A16MoEMethod:
    """FusedMoE method: AWQ int4 experts (group ``group_size``) on the sm_100a grouped GEMM."""

    pack_factor = 8  # int4 codes per int32

    def __init__(self, group_size: int = 128, weight_bits: int = 4, ep_group=None):
        if weight_bits != 4:
            raise ValueError("W4A16MoEMethod supports 4-bit weights only")
        if group_size != 128:
            raise ValueError("W4A16MoEMethod supports group size 128 only")
        self.group_size, self.weight_bits, self.ep_group = group_size, weight_bits, ep_group

    def create_weights(self, layer: torch.nn.Module, num_experts: int, hidden_size: int,
                       intermediate_size_per_partition: int, params_dtype: torch.dtype, **extra_weight_attrs):
        I, H, G, pf = intermediate_size_per_partition, hidden_size, self.group_size, self.pack_factor
        shapes = {
            "w13_qweight": ((num_experts, H, 2 * I // pf), torch.int32),
            "w2_qweight": ((num_experts, I, H // pf), torch.int32),
            "w13_scales": ((num_experts, H // G, 2 * I), params_dtype),
            "w2_scales": ((num_experts, I // G, H), params_dtype),
            "w13_qzeros": ((num_experts, H // G, 2 * I // pf), torch.int32),
            "w2_qzeros": ((num_experts, I // G, H // pf), torch.int32),
        }
        for name, (shape, dtype) in shapes.items():
            p = Parameter(torch.empty(shape, dtype=dtype), requires_grad=False)
            for k, v in extra_weight_attrs.items():
                setattr(p, k, v)
            layer.register_parameter(name, p)
        layer.num_groups_w13, layer.num_groups_w2 = H // G, I // G

    def process_weights_after_loading(self, layer: torch.nn.Module) -> None:
        """AWQ tensors -> packed blocks on their device; the AWQ parameters are released."""
        t = [getattr(layer, n).data for n in _AWQ_PARAMS]
        layer.w4a16_weights = pack_moe_awq(*t, group_size=self.group_size)
        for n in _AWQ_PARAMS:
            setattr(layer, n, Parameter(torch.empty(0, dtype=getattr(layer, n).dtype, device=t[0].device),
                                        requires_grad=False))

    def apply(self, layer: torch.nn.Module, x: torch.Tensor, topk_weights: torch.Tensor | None = None,
              topk_ids: torch.Tensor | None = None, *, router_logits: torch.Tensor | None = None,
              top_k: int | None = None, renormalize: bool = True, scoring_func: str = "softmax",
              num_expert_group: int = 0, topk_group: int = 0, e_score_correction_bias=None,
              routed_scaling_factor: float = 1.0, **_unused) -> torch.Tensor:
        """With routing already done (vLLM's current ``apply(layer, x, topk_weights, topk_ids, ...)``),
        or from router logits (``router_logits=, top_k=``, the older signature)."""
        w = layer.w4a16_weights
        if topk_ids is not None:
            return moe_w4a16(x, w, topk_weights, topk_ids, ep_group=self.ep_group)
        if router_logits is None or top_k is None:
            raise ValueError("apply needs (topk_weights, topk_ids) or (router_logits, top_k)")
        return fused_moe_w4a16(x, router_logits, w, top_k, scoring_func, renormalize, ep_group=self.ep_group,
                               num_expert_group=num_expert_group, topk_group=topk_group,
                               e_score_correction_bias=e_score_correction_bias,
                               routed_scaling_factor=routed_scaling_factor)
