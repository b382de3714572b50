"""ctypes binding of ``lib/libw4a16moe.so`` (the C ABI declared in ``include/w4a16_moe.h``).

There is no CPU fallback: if the library is missing or cannot be loaded every op raises
``W4A16Error`` loudly.
"""
from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent.parent / "lib" / "libw4a16moe.so"

W4_OK = 0
ERRORS = {
    -1: "W4_ERR_ARG (null pointer / bad enum)",
    -2: "W4_ERR_SHAPE (extent not tile-aligned or too large)",
    -3: "W4_ERR_DTYPE (unsupported activation dtype)",
    -4: "W4_ERR_GROUP (only group size 128 is supported)",
    -5: "W4_ERR_CUDA (launch / driver failure)",
    -6: "W4_ERR_WORKSPACE (workspace too small)",
    -7: "W4_ERR_NCCL (NCCL not loadable, or a collective failed)",
}
DTYPE_F16, DTYPE_BF16 = 0, 1
SCORE_SOFTMAX, SCORE_SIGMOID = 0, 1


class W4A16Error(RuntimeError):
    pass


_p, _i, _i64, _sz = C.c_void_p, C.c_int, C.c_int64, C.c_size_t

# name -> (restype, argtypes); must list every function of include/w4a16_moe.h
SIGNATURES = {
    "w4a16_packed_bytes": (_i64, [_i64, _i64, _i64]),
    "w4a16_tile_rows": (_i, []),
    "w4a16_tile_k": (_i, []),
    "w4a16_part_bytes": (_i, []),
    "w4a16_repack_awq": (_i, [_p, _p, _p, _i64, _i64, _i64, _i, _i, _p, _p]),
    "w4a16_dequant": (_i, [_p, _i64, _i64, _i64, _i, _i, _p, _p]),
    "w4a16_route_topk": (_i, [_p, _i64, _i64, _i64, _i, _i, _p, _p, _p]),
    "w4a16_route_grouped_topk": (_i, [_p, _i64, _i64, _i64, _i64, _i64, _i, _i, _p, C.c_float, _p, _p, _p]),
    "w4a16_route_permute": (_i, [_p, _i64, _i64, _i64, _i, _i, _p, _p, _p, _p, _p, _p, _p]),
    "w4a16_moe_permute": (_i, [_p, _i64, _i64, _p, _p, _p, _p, _p]),
    "w4a16_moe_permute_ws": (_i, [_p, _i64, _i64, _p, _p, _p, _p, _p, _i64, _p]),
    "w4a16_moe_permute_ws_bytes": (_i64, [_i64, _i64]),
    "w4a16_ep_local_order": (_i, [_p, _i64, _i64, _p, _p, _p, _p, _p]),
    "w4a16_moe_gather": (_i, [_p, _i64, _i64, _p, _i64, _p, _p, _p]),
    "w4a16_moe_combine": (_i, [_p, _i64, _i64, _i64, _p, _p, _i, _p, _p]),
    "w4a16_moe_gather_sums": (_i, [_p, _i64, _i64, _p, _i64, _p, _p, _i, _p, _p]),
    "w4a16_group_sums": (_i, [_p, _i64, _i64, _p, _i, _p, _p]),
    "w4a16_group_sums_ld": (_i64, [_i64]),
    "w4a16_grouped_gemm": (_i, [_p, _i64, _i64, _p, _i64, _i64, _i, _p, _p, _p, _p, _i, _i, _p]),
    "w4a16_pick_ntok": (_i, [_i64, _i64]),
    "w4a16_grouped_gemm_ws": (_i, [_p, _i64, _i64, _p, _i64, _i64, _i, _p, _p, _p, _p, _p, _p, _i, _i, _p, _i64,
                                   _p]),
    "w4a16_grouped_gemm_gather": (_i, [_p, _i64, _p, _i, _i64, _i64, _p, _i64, _i64, _i, _p, _p, _p, _p, _p, _i, _i,
                                       _p, _i64, _p]),
    "w4a16_grouped_gemm_ws_bytes": (_i64, [_i64, _i64, _i64, _i64, _i, _i]),
    "w4a16_decode_max_ntok": (_i, []),
    "w4a16_gemm_plan": (_i, [_i64, _i64, _i64, _i64, _i, _i, _i, _p, _p, _p, _p]),
    "w4a16_moe_workspace_bytes": (_i64, [_i64, _i64, _i64, _i64, _i64]),
    "w4a16_moe_forward": (_i, [_p, _i64, _i64, _i64, _i64, _i64, _p, _p, _p, _p, _i, _p, _p, _i64, _p]),
    "w4a16_moe_combine_f32": (_i, [_p, _i64, _i64, _i64, _p, _p, _i, _p, _p]),
    "w4a16_moe_forward_f32": (_i, [_p, _i64, _i64, _i64, _i64, _i64, _p, _p, _p, _p, _i, _p, _i, _p, _i64, _p]),
    "w4a16_ep_available": (_i, []),
    "w4a16_ep_unique_id": (_i, [_p]),
    "w4a16_ep_comm_init": (_i, [_p, _i, _i, _p]),
    "w4a16_ep_comm_wrap": (_i, [_p, _p]),
    "w4a16_ep_comm_destroy": (_i, [_p]),
    "w4a16_ep_comm_rank": (_i, [_p]),
    "w4a16_ep_comm_size": (_i, [_p]),
    "w4a16_ep_dispatch": (_i, [_p, _p, _p, _p, _i64, _i64, _i64, _i, _p, _p, _p, _p]),
    "w4a16_ep_localize": (_i, [_p, _i64, _i64, _i64, _p, _p]),
    "w4a16_ep_combine": (_i, [_p, _p, _i64, _i64, _i, _p, _p, _p]),
    "w4a16_moe_ep_workspace_bytes": (_i64, [_i64, _i64, _i64, _i64, _i64, _i64]),
    "w4a16_moe_forward_ep": (_i, [_p, _p, _i64, _i64, _i64, _i64, _i64, _p, _p, _p, _p, _i, _p, _p, _i64, _p]),
}
# debug aids exported by the library but not part of the public header
DEBUG_SIGNATURES = {
    "w4a16_debug_trace": (_i, [_p]),
    "w4a16_debug_trace_cta": (_i, [_i]),
    "w4a16_debug_stamp": (_i, [_p, _p]),
}

_lock = threading.Lock()
_lib = None


def load() -> C.CDLL:
    """Load (once) and return the library; raises W4A16Error when it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise W4A16Error(
                    f"{LIB_PATH} not built: run `python -m paper_2504_16214_b200._build` "
                    "(there is no CPU fallback for this path)")
            lib = C.CDLL(str(LIB_PATH))
            for name, (res, args) in {**SIGNATURES, **DEBUG_SIGNATURES}.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def check(rc: int, what: str) -> None:
    if rc != W4_OK:
        raise W4A16Error(f"{what} failed: {ERRORS.get(rc, rc)}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)
