"""AWQ checkpoints in, packed W4A16 expert blocks out (and back from disk).

* :func:`read_safetensors` / :func:`write_safetensors` -- the safetensors container (8-byte header
  length, JSON header of {name: {dtype, shape, data_offsets}}, raw little-endian payload), read into
  CPU tensors without the ``safetensors`` package (not in this image);
* :func:`stack_awq_experts` -- the per-expert AWQ tensors of one MoE layer as a HuggingFace AWQ
  checkpoint names them (``{prefix}.{e}.{gate_proj|up_proj|down_proj}.{qweight|qzeros|scales}``;
  Mixtral's ``w1 / w3 / w2`` via ``proj_names``) -> the six stacked tensors vLLM's AWQ MoE method
  holds (``w13_qweight [E, H, 2I/8]``, ``w13_scales [E, H/G, 2I]``, ``w13_qzeros [E, H/G, 2I/8]``,
  ``w2_*`` likewise with K = I), gate and up concatenated along N as vLLM does;
* :func:`save_packed` / :func:`load_packed` -- the repacked blocks on disk (a safetensors file whose
  metadata records the block-format version and the shapes), so serving loads them without the
  AWQ -> block repack.
"""
from __future__ import annotations

import json
import struct
from pathlib import Path

import torch

from .weights import MoEWeights, PackedW4, pack_moe_awq

BLOCK_FORMAT = "w4a16-blocks-v1"  # csrc/w4_format.cuh: 128x128 tiles, thread-major 16 B codes + scale/zero parts

_ST_DTYPES = {
    "I32": torch.int32, "F16": torch.float16, "BF16": torch.bfloat16, "F32": torch.float32, "U8": torch.uint8,
    "I64": torch.int64, "I8": torch.int8, "I16": torch.int16, "F64": torch.float64,
}
_ST_NAMES = {v: k for k, v in _ST_DTYPES.items()}


def read_safetensors(path) -> tuple[dict[str, torch.Tensor], dict[str, str]]:
    """(tensors on the CPU, the ``__metadata__`` strings) of one .safetensors file."""
    raw = Path(path).read_bytes()
    (n,) = struct.unpack("<Q", raw[:8])
    header = json.loads(raw[8:8 + n])
    meta = header.pop("__metadata__", {}) or {}
    base = 8 + n
    out = {}
    for name, info in header.items():
        if info["dtype"] not in _ST_DTYPES:
            raise ValueError(f"{name}: unsupported safetensors dtype {info['dtype']}")
        lo, hi = info["data_offsets"]
        buf = bytearray(raw[base + lo:base + hi])
        t = torch.frombuffer(buf, dtype=torch.uint8) if hi > lo else torch.empty(0, dtype=torch.uint8)
        out[name] = t.view(_ST_DTYPES[info["dtype"]]).reshape(info["shape"])
    return out, meta


def write_safetensors(path, tensors: dict[str, torch.Tensor], metadata: dict[str, str] | None = None) -> None:
    header: dict = {"__metadata__": dict(metadata or {})}
    blobs, at = [], 0
    for name in sorted(tensors):
        t = tensors[name].detach().contiguous().cpu()
        b = t.view(torch.uint8).numpy().tobytes() if t.numel() else b""
        header[name] = {"dtype": _ST_NAMES[t.dtype], "shape": list(t.shape), "data_offsets": [at, at + len(b)]}
        blobs.append(b)
        at += len(b)
    h = json.dumps(header, separators=(",", ":")).encode()
    h += b" " * (-len(h) % 8)  # 8-byte aligned payload
    with open(path, "wb") as f:
        f.write(struct.pack("<Q", len(h)))
        f.write(h)
        for b in blobs:
            f.write(b)


def stack_awq_experts(tensors: dict[str, torch.Tensor], prefix: str, num_experts: int,
                      proj_names=("gate_proj", "up_proj", "down_proj")) -> dict[str, torch.Tensor]:
    """Per-expert AWQ tensors -> vLLM's stacked ``w13_* / w2_*`` (gate | up concatenated on N)."""
    gate, up, down = proj_names

    def get(e, proj, what):
        key = f"{prefix}.{e}.{proj}.{what}"
        if key not in tensors:
            raise KeyError(f"checkpoint has no tensor {key!r}")
        return tensors[key]

    out = {}
    for what in ("qweight", "scales", "qzeros"):
        out[f"w13_{what}"] = torch.stack([torch.cat([get(e, gate, what), get(e, up, what)], dim=-1)
                                          for e in range(num_experts)])
        out[f"w2_{what}"] = torch.stack([get(e, down, what) for e in range(num_experts)])
    return out


def load_awq_moe(path_or_tensors, prefix: str, num_experts: int, device="cuda",
                 proj_names=("gate_proj", "up_proj", "down_proj"), group_size: int = 128) -> MoEWeights:
    """An AWQ MoE layer from a safetensors file (or an already-read tensor dict), packed on ``device``."""
    tensors = path_or_tensors if isinstance(path_or_tensors, dict) else read_safetensors(path_or_tensors)[0]
    s = stack_awq_experts(tensors, prefix, num_experts, proj_names)
    d = {k: v.to(device) for k, v in s.items()}
    return pack_moe_awq(d["w13_qweight"], d["w13_scales"], d["w13_qzeros"], d["w2_qweight"], d["w2_scales"],
                        d["w2_qzeros"], group_size)


def save_packed(path, weights: MoEWeights) -> None:
    """Packed blocks + shapes to disk (safetensors; metadata = block format and PackedW4 fields)."""
    meta = {"format": BLOCK_FORMAT}
    tensors = {}
    for name, pw in (("w13", weights.w13), ("w2", weights.w2)):
        tensors[f"{name}.blocks"] = pw.blocks
        meta[name] = json.dumps({"num_experts": pw.num_experts, "n_rows": pw.n_rows, "K": pw.K, "parts": pw.parts,
                                 "dtype": str(pw.dtype).replace("torch.", "")})
    write_safetensors(path, tensors, meta)


def load_packed(path, device="cuda") -> MoEWeights:
    tensors, meta = read_safetensors(path)
    if meta.get("format") != BLOCK_FORMAT:
        raise ValueError(f"{path}: not a {BLOCK_FORMAT} file (format {meta.get('format')!r})")
    parts = []
    for name in ("w13", "w2"):
        m = json.loads(meta[name])
        parts.append(PackedW4(tensors[f"{name}.blocks"].to(device), m["num_experts"], m["n_rows"], m["K"], m["parts"],
                              getattr(torch, m["dtype"])))
    return MoEWeights(*parts)
