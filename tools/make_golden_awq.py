#!/usr/bin/env python
"""Golden AWQ packing vectors from vLLM 0.22 (the third-party code whose conventions the numeric
oracle restates; see oracle/moe_oracle.py). Writes tests/golden/awq_pack_vllm.npz:
q [K, N] uint8 codes and vLLM's ``awq_pack(q, 4, K, N)`` int32 words (nibble interleave
0,2,4,6,1,3,5,7), plus the vLLM AWQ-triton reverse order used for unpacking."""
from pathlib import Path

import numpy as np
import torch
from vllm.model_executor.layers.quantization.utils.quant_utils import awq_pack

ROOT = Path(__file__).resolve().parent.parent


def main():
    rng = np.random.default_rng(20260417)
    out = {}
    for K, N in ((8, 8), (16, 64), (128, 256)):
        q = rng.integers(0, 16, size=(K, N), dtype=np.uint8)
        packed = awq_pack(torch.from_numpy(q.astype(np.int32)), 4, K, N).numpy()
        out[f"q_{K}x{N}"] = q
        out[f"packed_{K}x{N}"] = packed.astype(np.int32)
    np.savez_compressed(ROOT / "tests" / "golden" / "awq_pack_vllm.npz", **out)
    print(sorted(out))


if __name__ == "__main__":
    main()
