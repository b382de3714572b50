#!/usr/bin/env python
"""bench.py's other_configs (Llama dense linear, Mixtral / Qwen3 layers, Zipf routing) alone, one
compact line per config: for same-box A/B runs of build knobs (tools/gpu_ab_other.sh)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402

peaks = json.loads((Path(bench.__file__).parent / "MEASURED_PEAKS.json").read_text())
out = bench.other_configs(torch.device("cuda", 0), peaks["hbm_gbs"], peaks["bf16_tflops"])
for k, v in out.items():
    if isinstance(v, dict) and "ms" in v:
        xs = v.get("tokens", v.get("M", ""))
        print(f"  {k:34s} {xs} ms {v['ms']}")
