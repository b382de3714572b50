"""Packed W4A16 MoE weights: AWQ checkpoint tensors -> the kernel's block format (offline repack).

The block format (``csrc/w4_format.cuh``) is the "thread-major" repack the layout synthesizer
prescribes for the int4 operand (SURVEY.md Appendix A repack recipe; reference fixture
``/root/reference/pkg/fixtures/mixed_int4.prog:2-6``): each row-thread's 32 k-values are one
contiguous 16 B vector, so every int4 copy stays 16 B wide and the int4 -> fp16 cast needs no
inter-thread exchange. The byte count equals the AWQ payload exactly.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from . import ops


@dataclass(frozen=True)
class PackedW4:
    """One packed projection for all (local) experts."""
    blocks: torch.Tensor  # uint8 [num_experts * n_rows * K / 2 * (1 + 5/256)]
    num_experts: int
    n_rows: int           # output rows (2I for the fused gate/up projection)
    K: int                # reduction extent
    parts: int            # 2 = gate/up interleaved block-wise, 1 = plain
    dtype: torch.dtype    # activation (and scale) dtype

    @property
    def n_out(self) -> int:
        return self.n_rows // self.parts

    def dense(self) -> torch.Tensor:
        """Dequantised dense weights [E, n_rows, K] (test aid; runs the GEMM's dequantiser)."""
        return ops.dequant(self.blocks, self.num_experts, self.n_rows, self.K, self.parts, self.dtype)

    def slice_experts(self, start: int, stop: int) -> "PackedW4":
        per = self.blocks.numel() // self.num_experts
        return PackedW4(self.blocks[start * per:stop * per], stop - start, self.n_rows, self.K, self.parts,
                        self.dtype)


@dataclass(frozen=True)
class MoEWeights:
    w13: PackedW4  # gate/up: [E, 2I, H], parts = 2
    w2: PackedW4   # down:    [E, H, I],  parts = 1

    @property
    def num_experts(self) -> int:
        return self.w13.num_experts

    @property
    def hidden(self) -> int:
        return self.w13.K

    @property
    def inter(self) -> int:
        return self.w2.K

    def slice_experts(self, start: int, stop: int) -> "MoEWeights":
        return MoEWeights(self.w13.slice_experts(start, stop), self.w2.slice_experts(start, stop))


def pack_awq(qweight: torch.Tensor, scales: torch.Tensor, qzeros: torch.Tensor, gated: bool,
             group_size: int = 128) -> PackedW4:
    """AWQ tensors of one projection for all experts (``qweight [E, K, N/8] int32``,
    ``scales [E, K/G, N]`` in the activation dtype, ``qzeros [E, K/G, N/8] int32``) -> PackedW4.
    For ``gated`` the N rows are ``[gate (N/2) | up (N/2)]`` (vLLM's w13 layout)."""
    if qweight.dim() == 2:
        qweight, scales, qzeros = qweight[None], scales[None], qzeros[None]
    E, K, N8 = qweight.shape
    parts = 2 if gated else 1
    blocks = ops.repack_awq(qweight.contiguous(), scales.contiguous(), qzeros.contiguous(), parts, group_size)
    return PackedW4(blocks, E, N8 * 8, K, parts, scales.dtype)


def pack_moe_awq(w13_qweight, w13_scales, w13_qzeros, w2_qweight, w2_scales, w2_qzeros,
                 group_size: int = 128) -> MoEWeights:
    """vLLM AWQ MoE parameter set -> MoEWeights (w13: K = hidden, N = 2*inter; w2: K = inter,
    N = hidden)."""
    return MoEWeights(pack_awq(w13_qweight, w13_scales, w13_qzeros, True, group_size),
                      pack_awq(w2_qweight, w2_scales, w2_qzeros, False, group_size))


def random_moe_weights(E: int, H: int, I: int, dtype: torch.dtype, device="cuda", seed: int = 0) -> MoEWeights:
    """Synthetic AWQ weights of the named shapes generated on the device (q, z ~ U{0..15};
    scales ~ U(0.5, 1.5) * 2^-7), then packed. Used for benchmarks at full size."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)

    def one(N, K):
        qw = torch.randint(-2**31, 2**31 - 1, (E, K, N // 8), generator=g, device=device, dtype=torch.int64)
        qw = qw.to(torch.int32)
        qz = torch.randint(-2**31, 2**31 - 1, (E, K // 128, N // 8), generator=g, device=device,
                           dtype=torch.int64).to(torch.int32)
        sc = (torch.rand((E, K // 128, N), generator=g, device=device) + 0.5) * (2.0 ** -7)
        return qw, sc.to(dtype), qz

    a = one(2 * I, H)
    w13 = pack_awq(*a, gated=True)
    del a
    b = one(H, I)
    w2 = pack_awq(*b, gated=False)
    return MoEWeights(w13, w2)
