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

    def concat(self, other: "PackedW4") -> "PackedW4":
        """[self's experts | other's experts] (a copy; shapes and dtype must agree)."""
        if (self.n_rows, self.K, self.parts, self.dtype) != (other.n_rows, other.K, other.parts, other.dtype):
            raise ValueError("concat of packed weights with different shapes / dtype")
        return PackedW4(torch.cat([self.blocks, other.blocks]), self.num_experts + other.num_experts, self.n_rows,
                        self.K, self.parts, self.dtype)


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

    def concat(self, other: "MoEWeights") -> "MoEWeights":
        return MoEWeights(self.w13.concat(other.w13), self.w2.concat(other.w2))


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


def _expert_seed(seed: int, e: int, N: int, K: int) -> int:
    return (seed * 1_000_003 + e * 7919 + N * 131 + K) & 0x7FFF_FFFF_FFFF


def random_awq_expert(seed: int, e: int, N: int, K: int, dtype: torch.dtype, device="cuda"):
    """The synthetic AWQ tensors of expert ``e`` of a ``random_packed(..., generator=seed)`` projection
    (qweight [K, N/8] int32, scales [K/128, N], qzeros [K/128, N/8] int32): q, z ~ U{0..15} from random
    bytes, scales ~ U(0.5, 1.5) * 2^-7. Each expert has its own seed, so a checker can regenerate any
    sampled expert without the others."""
    g = torch.Generator(device=device)
    g.manual_seed(_expert_seed(seed, e, N, K))
    qw = torch.randint(0, 256, (K, N // 2), generator=g, device=device, dtype=torch.uint8).view(torch.int32)
    qz = torch.randint(0, 256, (K // 128, N // 2), generator=g, device=device, dtype=torch.uint8).view(torch.int32)
    sc = ((torch.rand((K // 128, N), generator=g, device=device) + 0.5) * (2.0 ** -7)).to(dtype)
    return qw, sc, qz


def random_packed(E: int, N: int, K: int, gated: bool, dtype: torch.dtype, generator, device="cuda",
                  chunk: int = 16) -> PackedW4:
    """Synthetic AWQ weights generated on the device and packed straight into one buffer.
    ``generator``: an int seed (per-expert streams, see :func:`random_awq_expert`) or a
    torch.Generator (expert chunks drawn from it in order)."""
    from . import _lib
    parts = 2 if gated else 1
    per = ops.packed_bytes(1, N, K)
    blocks = torch.empty(E * per, dtype=torch.uint8, device=device)
    if isinstance(generator, int):
        for e in range(E):
            qw, sc, qz = random_awq_expert(generator, e, N, K, dtype, device)
            _lib.call("w4a16_repack_awq", qw.data_ptr(), sc.data_ptr(), qz.data_ptr(), 1, K, N, parts, 128,
                      blocks[e * per:(e + 1) * per].data_ptr(), ops._stream())
        return PackedW4(blocks, E, N, K, parts, dtype)
    for e0 in range(0, E, chunk):
        n = min(chunk, E - e0)
        qw = torch.randint(0, 256, (n, K, N // 2), generator=generator, device=device,
                           dtype=torch.uint8).view(torch.int32)
        qz = torch.randint(0, 256, (n, K // 128, N // 2), generator=generator, device=device,
                           dtype=torch.uint8).view(torch.int32)
        sc = ((torch.rand((n, K // 128, N), generator=generator, device=device) + 0.5) * (2.0 ** -7)).to(dtype)
        out = blocks[e0 * per:(e0 + n) * per]
        _lib.call("w4a16_repack_awq", qw.data_ptr(), sc.data_ptr(), qz.data_ptr(), n, K, N, parts, 128,
                  out.data_ptr(), ops._stream())
        del qw, qz, sc
    return PackedW4(blocks, E, N, K, parts, dtype)


def random_moe_weights(E: int, H: int, I: int, dtype: torch.dtype, device="cuda", seed: int = 0) -> MoEWeights:
    """Synthetic packed MoE weights of the named shapes (benchmarks at full size). Expert e's AWQ
    tensors are ``random_awq_expert(2 * seed, e, 2 * I, H)`` (w13) and
    ``random_awq_expert(2 * seed + 1, e, H, I)`` (w2)."""
    return MoEWeights(random_packed(E, 2 * I, H, True, dtype, 2 * seed, device),
                      random_packed(E, H, I, False, dtype, 2 * seed + 1, device))
