#!/usr/bin/env python
"""Golden grouped top-k routing vectors from vLLM 0.22's torch ``grouped_topk`` (DeepSeek-V3/R1
routing; the reference has no routing code, see oracle/moe_oracle.py). Writes
tests/golden/grouped_topk_vllm.npz: per case the fp32 logits (and bias), vLLM's topk_ids sorted by
descending weight and the weights. Logits are drawn so that no two choices tie."""
import os
from pathlib import Path

import numpy as np
import torch

os.environ.setdefault("VLLM_USE_FUSED_MOE_GROUPED_TOPK", "0")
from vllm.model_executor.layers.fused_moe.router import grouped_topk_router  # noqa: E402

# the eager function under vLLM's @torch.compile wrapper (no inductor build needed on this host)
grouped_topk = grouped_topk_router.grouped_topk._torchdynamo_orig_callable

ROOT = Path(__file__).resolve().parent.parent
CASES = [  # name, T, E, k, groups, topk_group, scoring, renorm, bias, scale
    ("ds_r1", 64, 256, 8, 8, 4, "sigmoid", True, True, 2.5),
    ("ds_r1_nobias", 32, 256, 8, 8, 4, "sigmoid", True, False, 1.0),
    ("softmax_g4", 16, 64, 6, 4, 2, "softmax", False, False, 1.0),
    ("softmax_bias", 16, 128, 4, 8, 3, "softmax", True, True, 1.0),
]


def main():
    rng = np.random.default_rng(20261017)
    out = {}
    for name, T, E, k, G, TG, scoring, renorm, use_bias, scale in CASES:
        lg = rng.standard_normal((T, E)).astype(np.float32)
        bias = (rng.standard_normal(E) * 0.1).astype(np.float32) if use_bias else None
        w, ids = grouped_topk(torch.zeros((T, 1)), torch.from_numpy(lg), k, renorm, G, TG, scoring, scale,
                              torch.from_numpy(bias) if bias is not None else None)
        w, ids = w.numpy(), ids.numpy()
        order = np.argsort(-w, axis=1, kind="stable")  # vLLM's slot order is unspecified
        out[f"{name}_logits"] = lg
        if bias is not None:
            out[f"{name}_bias"] = bias
        out[f"{name}_ids"] = np.take_along_axis(ids, order, axis=1).astype(np.int32)
        out[f"{name}_weights"] = np.take_along_axis(w, order, axis=1).astype(np.float32)
        out[f"{name}_meta"] = np.array([T, E, k, G, TG, scoring == "softmax", renorm, use_bias], dtype=np.int64)
        out[f"{name}_scale"] = np.array([scale], dtype=np.float32)
    np.savez_compressed(ROOT / "tests" / "golden" / "grouped_topk_vllm.npz", **out)
    print(sorted(out))


if __name__ == "__main__":
    main()
