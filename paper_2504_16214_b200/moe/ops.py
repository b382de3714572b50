"""torch-tensor wrappers over the C ABI: each op validates, allocates outputs and launches on the
current CUDA stream. Inputs must already be CUDA tensors; nothing here runs on the CPU."""
from __future__ import annotations

import ctypes as C

import torch

from . import _lib

_ACT = {torch.float16: _lib.DTYPE_F16, torch.bfloat16: _lib.DTYPE_BF16}


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _need_cuda(*ts: torch.Tensor) -> None:
    for t in ts:
        if not t.is_cuda:
            raise _lib.W4A16Error("W4A16 ops take CUDA tensors (no CPU fallback)")
        if not t.is_contiguous():
            raise _lib.W4A16Error("W4A16 ops take contiguous tensors")


def act_code(dtype: torch.dtype) -> int:
    try:
        return _ACT[dtype]
    except KeyError:
        raise _lib.W4A16Error(f"activation dtype must be float16 or bfloat16, got {dtype}") from None


# ------------------------------------------------------------------------------------------ weights
def packed_bytes(num_experts: int, n_rows: int, K: int) -> int:
    n = _lib.load().w4a16_packed_bytes(num_experts, n_rows, K)
    if n < 0:
        raise _lib.W4A16Error(f"n_rows={n_rows} and K={K} must be multiples of 128")
    return n


def repack_awq(qweight: torch.Tensor, scales: torch.Tensor, qzeros: torch.Tensor, parts: int,
               group_size: int = 128) -> torch.Tensor:
    """AWQ [E][K][N/8] int32 / [E][K/G][N] / [E][K/G][N/8] -> packed uint8 blocks."""
    _need_cuda(qweight, scales, qzeros)
    E, K, N8 = qweight.shape
    N = N8 * 8
    if scales.shape != (E, K // group_size, N) or qzeros.shape != (E, K // group_size, N8):
        raise _lib.W4A16Error("AWQ scales/qzeros shapes do not match qweight")
    out = torch.empty(packed_bytes(E, N, K), dtype=torch.uint8, device=qweight.device)
    _lib.call("w4a16_repack_awq", qweight.data_ptr(), scales.data_ptr(), qzeros.data_ptr(), E, K, N, parts,
              group_size, out.data_ptr(), _stream())
    return out


def dequant(blocks: torch.Tensor, num_experts: int, n_rows: int, K: int, parts: int,
            dtype: torch.dtype) -> torch.Tensor:
    _need_cuda(blocks)
    out = torch.empty((num_experts, n_rows, K), dtype=dtype, device=blocks.device)
    _lib.call("w4a16_dequant", blocks.data_ptr(), num_experts, n_rows, K, parts, act_code(dtype), out.data_ptr(),
              _stream())
    return out


# ------------------------------------------------------------------------------------------ routing
def route_topk(logits: torch.Tensor, k: int, scoring: str = "softmax", renormalize: bool = False):
    _need_cuda(logits)
    if logits.dtype != torch.float32:
        raise _lib.W4A16Error("router logits must be float32")
    T, E = logits.shape
    ids = torch.empty((T, k), dtype=torch.int32, device=logits.device)
    wts = torch.empty((T, k), dtype=torch.float32, device=logits.device)
    sc = {"softmax": _lib.SCORE_SOFTMAX, "sigmoid": _lib.SCORE_SIGMOID}[scoring]
    _lib.call("w4a16_route_topk", logits.data_ptr(), T, E, k, sc, int(renormalize), ids.data_ptr(), wts.data_ptr(),
              _stream())
    return ids, wts


def route_permute(logits: torch.Tensor, k: int, scoring: str = "softmax", renormalize: bool = False):
    """route_topk + moe_permute of its ids in one single-CTA kernel (small batches).
    -> (ids, weights, expert_counts, expert_offsets, sorted_pairs, pair_pos)."""
    _need_cuda(logits)
    if logits.dtype != torch.float32:
        raise _lib.W4A16Error("router logits must be float32")
    T, E = logits.shape
    dev = logits.device
    ids = torch.empty((T, k), dtype=torch.int32, device=dev)
    wts = torch.empty((T, k), dtype=torch.float32, device=dev)
    counts = torch.empty(E, dtype=torch.int32, device=dev)
    offsets = torch.empty(E + 1, dtype=torch.int32, device=dev)
    sp = torch.empty(T * k, dtype=torch.int32, device=dev)
    pp = torch.empty(T * k, dtype=torch.int32, device=dev)
    sc = {"softmax": _lib.SCORE_SOFTMAX, "sigmoid": _lib.SCORE_SIGMOID}[scoring]
    _lib.call("w4a16_route_permute", logits.data_ptr(), T, E, k, sc, int(renormalize), ids.data_ptr(), wts.data_ptr(),
              counts.data_ptr(), offsets.data_ptr(), sp.data_ptr(), pp.data_ptr(), _stream())
    return ids, wts, counts, offsets, sp, pp


def route_grouped_topk(logits: torch.Tensor, k: int, num_groups: int, topk_group: int, scoring: str = "sigmoid",
                       renormalize: bool = True, bias: torch.Tensor | None = None,
                       routed_scaling_factor: float = 1.0):
    """DeepSeek-V3/R1 grouped top-k (vLLM ``grouped_topk`` semantics, see the C header)."""
    _need_cuda(logits)
    if logits.dtype != torch.float32:
        raise _lib.W4A16Error("router logits must be float32")
    T, E = logits.shape
    if bias is not None:
        _need_cuda(bias)
        bias = bias.float().contiguous()
        if bias.numel() != E:
            raise _lib.W4A16Error("e_score_correction_bias must have one entry per expert")
    ids = torch.empty((T, k), dtype=torch.int32, device=logits.device)
    wts = torch.empty((T, k), dtype=torch.float32, device=logits.device)
    sc = {"softmax": _lib.SCORE_SOFTMAX, "sigmoid": _lib.SCORE_SIGMOID}[scoring]
    _lib.call("w4a16_route_grouped_topk", logits.data_ptr(), T, E, k, num_groups, topk_group, sc, int(renormalize),
              bias.data_ptr() if bias is not None else None, float(routed_scaling_factor), ids.data_ptr(),
              wts.data_ptr(), _stream())
    return ids, wts


def moe_permute(topk_ids: torch.Tensor, num_experts: int, workspace: torch.Tensor | None = None):
    """-> (expert_counts [E], expert_offsets [E+1], sorted_pairs [P], pair_pos [P]) int32. Large P runs
    the multi-CTA kernel when a workspace of permute_ws_bytes(P, E) bytes is given (or allocated)."""
    _need_cuda(topk_ids)
    if topk_ids.dtype != torch.int32:
        raise _lib.W4A16Error("topk_ids must be int32")
    P = topk_ids.numel()
    dev = topk_ids.device
    counts = torch.empty(num_experts, dtype=torch.int32, device=dev)
    offsets = torch.empty(num_experts + 1, dtype=torch.int32, device=dev)
    sorted_pairs = torch.empty(max(P, 1), dtype=torch.int32, device=dev)
    pair_pos = torch.empty(max(P, 1), dtype=torch.int32, device=dev)
    wsb = permute_ws_bytes(P, num_experts)
    if workspace is None or workspace.numel() * workspace.element_size() < wsb:
        workspace = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
    _lib.call("w4a16_moe_permute_ws", topk_ids.data_ptr(), P, num_experts, counts.data_ptr(), offsets.data_ptr(),
              sorted_pairs.data_ptr(), pair_pos.data_ptr(), workspace.data_ptr(),
              workspace.numel() * workspace.element_size(), _stream())
    return counts, offsets, sorted_pairs[:P], pair_pos[:P]


def permute_ws_bytes(P: int, num_experts: int) -> int:
    return int(_lib.load().w4a16_moe_permute_ws_bytes(P, num_experts))


def moe_gather(x: torch.Tensor, sorted_pairs: torch.Tensor, topk: int, rows: int | None = None,
               row_limit: torch.Tensor | None = None, out: torch.Tensor | None = None) -> torch.Tensor:
    _need_cuda(x, sorted_pairs)
    act_code(x.dtype)
    rows = sorted_pairs.numel() if rows is None else rows
    H = x.shape[1]
    if out is None:
        out = torch.empty((rows, H), dtype=x.dtype, device=x.device)
    _lib.call("w4a16_moe_gather", x.data_ptr(), H, topk, sorted_pairs.data_ptr(), rows, _ptr(row_limit),
              out.data_ptr(), _stream())
    return out


def ep_local_order(recv_counts: torch.Tensor, n_recv: int):
    """recv_counts [world, E_l] int32 (device) -> (l_counts [E_l], l_offsets [E_l+1], l_sorted [n],
    l_pos [n]) int32: the received rows' local-expert order (see include/w4a16_moe.h)."""
    _need_cuda(recv_counts)
    world, el = recv_counts.shape
    dev = recv_counts.device
    l_counts = torch.empty(el, dtype=torch.int32, device=dev)
    l_offsets = torch.empty(el + 1, dtype=torch.int32, device=dev)
    l_sorted = torch.empty(max(n_recv, 1), dtype=torch.int32, device=dev)
    l_pos = torch.empty(max(n_recv, 1), dtype=torch.int32, device=dev)
    _lib.call("w4a16_ep_local_order", recv_counts.contiguous().data_ptr(), world, el, l_counts.data_ptr(),
              l_offsets.data_ptr(), l_sorted.data_ptr(), l_pos.data_ptr(), _stream())
    return l_counts, l_offsets, l_sorted[:n_recv], l_pos[:n_recv]


def sums_shape(rows: int, K: int) -> tuple[int, int, int]:
    """Shape of the per-(k-group, row) activation sums array: [K/128][ld][2] fp32."""
    return (K // 128, int(_lib.load().w4a16_group_sums_ld(rows)), 2)


def moe_gather_sums(x: torch.Tensor, sorted_pairs: torch.Tensor, topk: int, rows: int | None = None,
                    row_limit: torch.Tensor | None = None, out: torch.Tensor | None = None,
                    sums: torch.Tensor | None = None) -> tuple[torch.Tensor, torch.Tensor]:
    """moe_gather plus the (C, S) group sums of the gathered rows (decode-mode GEMM input)."""
    _need_cuda(x, sorted_pairs)
    rows = sorted_pairs.numel() if rows is None else rows
    H = x.shape[1]
    if out is None:
        out = torch.empty((rows, H), dtype=x.dtype, device=x.device)
    if sums is None:
        sums = torch.empty(sums_shape(rows, H), dtype=torch.float32, device=x.device)
    _lib.call("w4a16_moe_gather_sums", x.data_ptr(), H, topk, sorted_pairs.data_ptr(), rows, _ptr(row_limit),
              out.data_ptr(), act_code(x.dtype), sums.data_ptr(), _stream())
    return out, sums


def group_sums(x: torch.Tensor, row_limit: torch.Tensor | None = None,
               out: torch.Tensor | None = None) -> torch.Tensor:
    """(C, S) sums per (k-group of 128, row) of x [rows, K] (see include/w4a16_moe.h)."""
    _need_cuda(x)
    rows, K = x.shape
    if out is None:
        out = torch.empty(sums_shape(rows, K), dtype=torch.float32, device=x.device)
    _lib.call("w4a16_group_sums", x.data_ptr(), rows, K, _ptr(row_limit), act_code(x.dtype), out.data_ptr(),
              _stream())
    return out


def moe_combine(y_perm: torch.Tensor, pair_pos: torch.Tensor, topk_weights: torch.Tensor,
                out: torch.Tensor | None = None, f32: bool = False) -> torch.Tensor:
    """y[t] = act(sum_j w[t, j] Y[pos(t, j)]) -- or, with ``f32``, the fp32 sums unrounded (float32
    output: the expert-parallel partial)."""
    _need_cuda(y_perm, pair_pos, topk_weights)
    T, k = topk_weights.shape
    H = y_perm.shape[1]
    if out is None:
        out = torch.empty((T, H), dtype=torch.float32 if f32 else y_perm.dtype, device=y_perm.device)
    _lib.call("w4a16_moe_combine_f32" if f32 else "w4a16_moe_combine", y_perm.data_ptr(), T, H, k, pair_pos.data_ptr(),
              topk_weights.data_ptr(), act_code(y_perm.dtype), out.data_ptr(), _stream())
    return out


# ------------------------------------------------------------------------------- expert parallelism
def ep_available() -> bool:
    return bool(_lib.load().w4a16_ep_available())


def ep_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _lib.call("w4a16_ep_unique_id", C.addressof(buf))
    return bytes(buf)


def ep_comm_init(uid: bytes, rank: int, world: int) -> int:
    """Opaque communicator handle (an int address) over ``world`` ranks; collective."""
    buf = (C.c_uint8 * 128).from_buffer_copy(uid)
    out = C.c_void_p()
    _lib.call("w4a16_ep_comm_init", C.addressof(buf), rank, world, C.byref(out))
    return out.value


def ep_comm_destroy(comm: int) -> None:
    _lib.call("w4a16_ep_comm_destroy", comm)


def ep_dispatch(comm: int, world: int, x: torch.Tensor, topk_ids: torch.Tensor, topk_weights: torch.Tensor,
                out: tuple | None = None):
    """All-gather (x, ids, weights) of every rank -> ([world*T, H], [world*T, k], [world*T, k])."""
    _need_cuda(x, topk_ids, topk_weights)
    T, H = x.shape
    k = topk_ids.shape[1]
    x_all, ids_all, w_all = out or (x.new_empty((world * T, H)), topk_ids.new_empty((world * T, k)),
                                    topk_weights.new_empty((world * T, k)))
    _lib.call("w4a16_ep_dispatch", comm, x.data_ptr(), topk_ids.data_ptr(), topk_weights.data_ptr(), T, H, k,
              act_code(x.dtype), x_all.data_ptr(), ids_all.data_ptr(), w_all.data_ptr(), _stream())
    return x_all, ids_all, w_all


def ep_localize(ids: torch.Tensor, expert_base: int, local_experts: int, out: torch.Tensor | None = None):
    _need_cuda(ids)
    out = torch.empty_like(ids) if out is None else out
    _lib.call("w4a16_ep_localize", ids.data_ptr(), ids.numel(), expert_base, local_experts, out.data_ptr(), _stream())
    return out


def ep_combine(comm: int, partial: torch.Tensor, T: int, dtype: torch.dtype, reduced: torch.Tensor | None = None,
               out: torch.Tensor | None = None) -> torch.Tensor:
    """Reduce-scatter the fp32 partials [world*T, H] (sum over ranks) -> act(dtype) [T, H]."""
    _need_cuda(partial)
    H = partial.shape[1]
    reduced = partial.new_empty((T, H)) if reduced is None else reduced
    out = torch.empty((T, H), dtype=dtype, device=partial.device) if out is None else out
    _lib.call("w4a16_ep_combine", comm, partial.data_ptr(), T, H, act_code(dtype), reduced.data_ptr(), out.data_ptr(),
              _stream())
    return out


# ------------------------------------------------------------------------------------------ GEMM
def grouped_gemm(x: torch.Tensor, blocks: torch.Tensor, num_experts: int, n_out: int, gated: bool,
                 expert_counts: torch.Tensor, expert_offsets: torch.Tensor, ntok: int = 0,
                 out: torch.Tensor | None = None, xsum: torch.Tensor | None = None,
                 workspace: torch.Tensor | None = None, osum: torch.Tensor | None = None,
                 out_rows: torch.Tensor | None = None) -> torch.Tensor:
    """out[off_e + m] = act(x[off_e + m] @ W_e^T) (gated: silu(gate) * up), per expert. ``xsum``
    (group_sums / moe_gather_sums of x) selects the decode kernel for 16/32-token tiles; a
    ``workspace`` of gemm_ws_bytes(...) bytes enables split-K when few tiles exist; ``osum`` (shape
    sums_shape(rows, n_out)) receives the output's group sums (the next GEMM's xsum); ``out_rows``
    (int32 [rows]) scatters result row i to out row out_rows[i]."""
    _need_cuda(x, blocks, expert_counts, expert_offsets)
    rows, K = x.shape
    if out is None:
        out = torch.empty((rows, n_out), dtype=x.dtype, device=x.device)
    wsb = 0 if workspace is None else workspace.numel() * workspace.element_size()
    _lib.call("w4a16_grouped_gemm_ws", x.data_ptr(), rows, K, blocks.data_ptr(), num_experts, n_out, int(gated),
              expert_counts.data_ptr(), expert_offsets.data_ptr(), _ptr(xsum), _ptr(osum), _ptr(out_rows),
              out.data_ptr(), act_code(x.dtype), ntok, _ptr(workspace), wsb, _stream())
    return out


def grouped_gemm_gather(x: torch.Tensor, gather_rows: torch.Tensor, gather_div: int, blocks: torch.Tensor,
                        num_experts: int, n_out: int, gated: bool, expert_counts: torch.Tensor,
                        expert_offsets: torch.Tensor, ntok: int = 0, out: torch.Tensor | None = None,
                        xsum: torch.Tensor | None = None, workspace: torch.Tensor | None = None,
                        osum: torch.Tensor | None = None, rows: int | None = None) -> torch.Tensor:
    """grouped_gemm on the rows x[gather_rows[i] // gather_div] (i < rows) without materialising them:
    the GEMM's producer gathers them with TMA gather4. ``xsum`` = group_sums(x) (x's own rows)."""
    _need_cuda(x, gather_rows, blocks, expert_counts, expert_offsets)
    if gather_rows.dtype != torch.int32:
        raise _lib.W4A16Error("gather_rows must be int32")
    rows = gather_rows.numel() if rows is None else rows
    x_rows, K = x.shape
    if out is None:
        out = torch.empty((rows, n_out), dtype=x.dtype, device=x.device)
    wsb = 0 if workspace is None else workspace.numel() * workspace.element_size()
    _lib.call("w4a16_grouped_gemm_gather", x.data_ptr(), x_rows, gather_rows.data_ptr(), gather_div, rows, K,
              blocks.data_ptr(), num_experts, n_out, int(gated), expert_counts.data_ptr(), expert_offsets.data_ptr(),
              _ptr(xsum), _ptr(osum), out.data_ptr(), act_code(x.dtype), ntok, _ptr(workspace), wsb, _stream())
    return out


def decode_max_ntok() -> int:
    """Largest token tile the grouped GEMM runs in offset-code (decode) mode (W4A16_DECODE_MAX_NTOK)."""
    return int(_lib.load().w4a16_decode_max_ntok())


def gemm_ws_bytes(rows: int, K: int, num_experts: int, n_out: int, gated: bool, ntok: int = 0) -> int:
    """Split-K workspace bytes the decode-mode grouped GEMM would use (0: no split planned)."""
    return int(_lib.load().w4a16_grouped_gemm_ws_bytes(rows, K, num_experts, n_out, int(gated), ntok))


def pick_ntok(rows: int, num_experts: int) -> int:
    return _lib.load().w4a16_pick_ntok(rows, num_experts)
