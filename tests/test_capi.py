"""C ABI boundary checks that need no GPU: the in-tree library loads and exports every function
declared in include/*.h, and the host wrappers declare a signature for each of them."""
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _declared():
    names = set()
    for h in (ROOT / "include").glob("*.h"):
        text = re.sub(r"/\*.*?\*/", "", h.read_text(), flags=re.S)
        names |= set(re.findall(r"\b(w4a16_\w+)\s*\(", text))
    return names


def test_header_declares_the_path():
    d = _declared()
    for fn in ("w4a16_grouped_gemm", "w4a16_route_topk", "w4a16_route_grouped_topk", "w4a16_route_permute", "w4a16_moe_permute", "w4a16_moe_gather",
               "w4a16_moe_combine", "w4a16_repack_awq", "w4a16_dequant", "w4a16_moe_forward"):
        assert fn in d


def test_library_exports_every_declared_symbol():
    from paper_2504_16214_b200 import _build
    from paper_2504_16214_b200.moe import _lib
    _build.build()
    lib = _lib.load()
    missing = [n for n in sorted(_declared()) if not hasattr(lib, n)]
    assert not missing, missing
    assert set(_lib.SIGNATURES) == _declared()


def test_pure_host_queries():
    from paper_2504_16214_b200.moe import _lib
    lib = _lib.load()
    assert lib.w4a16_tile_rows() == 128 and lib.w4a16_tile_k() == 128
    # packed bytes == AWQ payload bytes (codes + fp16 scales + int4 zeros)
    E, N, K = 256, 4096, 7168
    assert lib.w4a16_packed_bytes(E, N, K) == E * (N * K // 2 + (K // 128) * N * 2 + (K // 128) * N // 2)
    assert lib.w4a16_packed_bytes(1, 100, 128) == -1
    assert lib.w4a16_pick_ntok(512, 256) == 16 and lib.w4a16_pick_ntok(65536, 256) == 128


def test_ops_refuse_cpu_tensors():
    torch = pytest.importorskip("torch")
    from paper_2504_16214_b200.moe import _lib, ops
    with pytest.raises(_lib.W4A16Error):
        ops.moe_permute(torch.zeros(8, dtype=torch.int32), 4)


def test_token_tile_choice():
    """w4a16_pick_ntok at the points tools/ntok_probe.py measured (whole-layer time per tile size):
    the expected-m-tiles cost model picks the measured-fastest tile for each MoE case; one dense
    matrix keeps the mean + 2.5 sigma rule (its full 16-token offset tiles measured slower)."""
    from paper_2504_16214_b200.moe import _lib
    lib = _lib.load()
    picks = {  # (rows = T * k, experts) -> measured-best tile
        (96, 8): 16,      # Mixtral T=48
        (384, 8): 64,     # Mixtral T=192
        (128, 8): 32,     # Mixtral T=64 (32 and 64 measured equal)
        (2048, 128): 32,  # Qwen3 T=256
        (1536, 128): 16,  # Qwen3 T=192
        (4096, 256): 32,  # DS-R1 T=512
        (512, 256): 16,   # DS-R1 T=64
        (65536, 256): 128,
        (16, 1): 32,      # dense M=16
        (1, 1): 16,
    }
    for (rows, e), want in picks.items():
        assert lib.w4a16_pick_ntok(rows, e) == want, (rows, e)


def test_gemm_plan_rules():
    """The planner's block-mode rules (w4a16_gemm_plan, no GPU): decode down projections use n-pair
    stages unless an upper estimate of the n-pair tiles leaves SMs idle (k-pair then); 128-token
    prefill down projections of short K use plain stages; 64-token ones n-pair (sm_count() is 148
    when no GPU is visible, as on a B200)."""
    import ctypes
    from paper_2504_16214_b200.moe import _lib
    lib = _lib.load()
    f = lib.w4a16_gemm_plan
    f.restype = ctypes.c_int
    f.argtypes = [ctypes.c_int64] * 4 + [ctypes.c_int] * 3 + [ctypes.POINTER(ctypes.c_int)] * 4

    def plan(rows, K, E, N, gated, xsum, ntok=0):
        o = [ctypes.c_int() for _ in range(4)]
        assert f(rows, K, E, N, gated, xsum, ntok, *[ctypes.byref(v) for v in o]) == 0
        return tuple(v.value for v in o)  # (ntok, mode, offset, splits)

    PLAIN, GATEUP, KPAIR, NPAIR = 0, 1, 2, 3
    assert plan(512, 2048, 256, 7168, 0, 1)[:3] == (16, NPAIR, 1)   # DS-R1 T=64 down: decode n-pair
    assert plan(8, 2048, 256, 7168, 0, 1)[1] == NPAIR               # DS-R1 T=1 down: 224 n-pair tiles
    assert plan(8, 768, 128, 2048, 0, 1)[1] == KPAIR                # Qwen3 T=1 down: 64 n-pair tiles < 148
    assert plan(2, 14336, 8, 4096, 0, 1)[1] == KPAIR                # Mixtral T=1 down
    assert plan(512, 7168, 256, 2048, 1, 1)[:3] == (16, GATEUP, 1)  # DS-R1 T=64 gate/up
    assert plan(65536, 2048, 256, 7168, 0, 0)[:3] == (128, NPAIR, 0)  # DS-R1 prefill down (K/128 = 16)
    assert plan(65536, 768, 128, 2048, 0, 0)[:3] == (128, PLAIN, 0)   # Qwen3 prefill down (K/128 = 6)
    assert plan(8192, 2048, 256, 7168, 0, 0)[:2] == (64, NPAIR)       # DS-R1 T=1024 down: 64-token n-pair
