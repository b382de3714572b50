"""Expert parallelism: experts sharded contiguously across the ranks of one node, tokens exchanged
by all-to-all(v) over NCCL (NVLink / NVSwitch) for dispatch and combine.

Rank r owns global experts [r*E_l, (r+1)*E_l). Each rank routes its own tokens, then:

  1. permute its (token, slot) pairs by *global* expert (stable counting sort, CUDA) -- this also
     groups them by destination rank, since experts are contiguous per rank;
  2. gather the rows (CUDA) into the send buffer;
  3. exchange per-expert counts (all_to_all_single, int32 [world * E_l]) and read the split sizes
     back to the host (the one host synchronisation EP needs: NCCL all-to-all-v takes host splits);
  4. all_to_all_single the rows (dispatch);
  5. received rows arrive grouped by (source rank, local expert); permute them by local expert
     (CUDA) and run the two grouped GEMMs on the local shard;
  6. un-permute back to arrival order, all_to_all_single back (combine), and reduce the k expert
     outputs of every token with its routing weights (CUDA).

The only collective is the exchange step itself. ``backend`` supplies the primitive
ops; the product path uses the CUDA ops (:mod:`.ops`) -- tests inject a CPU backend to exercise the
exchange plumbing on ``gloo`` with world_size 2.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import ops as cuda_ops


@dataclass
class DispatchPlan:
    send_splits: list[int]      # rows this rank sends to each rank
    recv_splits: list[int]      # rows this rank receives from each rank
    recv_counts: torch.Tensor   # [world, E_l] int32: rows per (source rank, local expert)


def plan_dispatch(global_counts: torch.Tensor, world: int, group=None) -> DispatchPlan:
    """global_counts [world * E_l] int32 (rows this rank routes to each global expert)."""
    e_local = global_counts.numel() // world
    recv = torch.empty_like(global_counts)
    dist.all_to_all_single(recv, global_counts.contiguous(), group=group)
    send_splits = global_counts.view(world, e_local).sum(dim=1)
    both = torch.cat([send_splits, recv.view(world, e_local).sum(dim=1)]).cpu().tolist()
    return DispatchPlan(both[:world], both[world:], recv.view(world, e_local))


def local_expert_ids(recv_counts: torch.Tensor, n_recv: int | None = None) -> torch.Tensor:
    """Local expert id of every received row (rows arrive grouped by source, then by expert).
    ``n_recv`` (the host-known total) avoids a device->host synchronisation."""
    world, e_local = recv_counts.shape
    experts = torch.arange(e_local, device=recv_counts.device, dtype=torch.int32).repeat(world)
    return torch.repeat_interleave(experts, recv_counts.reshape(-1).to(torch.int64),
                                   output_size=n_recv).to(torch.int32)


class CudaBackend:
    permute = staticmethod(cuda_ops.moe_permute)
    local_order = staticmethod(cuda_ops.ep_local_order)  # one kernel: receiver-side local expert order
    scatter_out = True  # the down GEMM writes arrival order directly
    gather = staticmethod(cuda_ops.moe_gather)
    combine = staticmethod(cuda_ops.moe_combine)

    @staticmethod
    def experts(x, weights, counts, offsets, ntok, timer=None, out_rows=None):
        """Both grouped GEMMs; with ``out_rows`` the down projection writes its rows scattered
        through it (straight back to arrival order)."""
        from .layer import _NOTIMER
        tm = timer or _NOTIMER
        E, H, I = weights.num_experts, weights.hidden, weights.inter
        nt = ntok or cuda_ops.pick_ntok(x.shape[0], E)
        from .layer import _DECODE_MAX_NTOK
        decode = nt <= _DECODE_MAX_NTOK
        xs = hs = None
        if decode:
            with tm.span("sums_x"):
                xs = cuda_ops.group_sums(x)
        with tm.span("gemm_gate_up"):
            h = cuda_ops.grouped_gemm(x, weights.w13.blocks, E, I, True, counts, offsets, nt, xsum=xs)
        if decode:
            with tm.span("sums_h"):
                hs = cuda_ops.group_sums(h)
        with tm.span("gemm_down"):
            return cuda_ops.grouped_gemm(h, weights.w2.blocks, E, H, False, counts, offsets, nt, xsum=hs,
                                         out_rows=out_rows)


def moe_w4a16_ep(x: torch.Tensor, weights, topk_weights: torch.Tensor, topk_ids: torch.Tensor, group=None,
                 ntok: int = 0, timer=None, backend=CudaBackend) -> torch.Tensor:
    """Expert-parallel W4A16 MoE. ``weights`` holds this rank's contiguous expert shard;
    ``topk_ids`` are global expert ids."""
    world = dist.get_world_size(group)
    T, H = x.shape
    k = topk_ids.shape[1]
    e_local = weights.num_experts
    e_global = e_local * world
    topk_ids = topk_ids.to(torch.int32).contiguous()
    topk_weights = topk_weights.to(torch.float32).contiguous()

    from .layer import _NOTIMER
    tm = timer or _NOTIMER
    # 1-2: group pairs by destination (global expert order) and pack rows
    with tm.span("permute"):
        g_counts, g_offsets, sorted_pairs, pair_pos = backend.permute(topk_ids, e_global)
    with tm.span("gather"):
        # row_limit = the number of valid pairs (ids < 0 or >= e_global are dropped by the permutation
        # and leave the tail of sorted_pairs unwritten): the gather never reads those entries
        send_x = backend.gather(x.contiguous(), sorted_pairs, k, T * k, g_offsets[e_global:])
    # 3: counts exchange + host splits
    plan = plan_dispatch(g_counts, world, group)
    n_recv = sum(plan.recv_splits)
    # 4: dispatch
    recv_x = x.new_empty((n_recv, H))
    dist.all_to_all_single(recv_x, send_x, plan.recv_splits, plan.send_splits, group=group)
    # 5: local expert order + grouped GEMMs
    if hasattr(backend, "local_order"):
        with tm.span("local_order"):
            l_counts, l_offsets, l_sorted, l_pos = backend.local_order(plan.recv_counts, n_recv)
    else:  # generic: ids of the received rows, then the stable permutation
        lid = local_expert_ids(plan.recv_counts, n_recv)
        l_counts, l_offsets, l_sorted, l_pos = backend.permute(lid, e_local)
    with tm.span("gather_local"):
        xl = backend.gather(recv_x, l_sorted, 1, n_recv) if n_recv else recv_x
    # 6: the down GEMM scatters its rows straight back to arrival order; combine exchange, reduction
    if not n_recv:
        y_recv = recv_x
    elif getattr(backend, "scatter_out", False):
        y_recv = backend.experts(xl, weights, l_counts, l_offsets, ntok, timer, out_rows=l_sorted)
    else:
        yl = backend.experts(xl, weights, l_counts, l_offsets, ntok, timer)
        y_recv = backend.gather(yl, l_pos, 1, n_recv)
    y_back = x.new_empty((T * k, H))
    dist.all_to_all_single(y_back, y_recv, plan.send_splits, plan.recv_splits, group=group)
    with tm.span("combine"):
        return backend.combine(y_back, pair_pos, topk_weights)


def shard_with_shared(weights, num_shared: int, world: int, rank: int):
    """Full packed weights laid out [routed experts | shared experts] -> (this rank's contiguous
    routed shard, the shared experts), the two pieces ``fused_moe_w4a16(..., ep_group=...,
    shared_weights=...)`` takes. The shared experts are replicated on every rank."""
    routed = weights.num_experts - num_shared
    lo, hi = shard_bounds(routed, world, rank)
    return weights.slice_experts(lo, hi), weights.slice_experts(routed, weights.num_experts)


def shard_bounds(num_experts: int, world: int, rank: int) -> tuple[int, int]:
    if num_experts % world:
        raise ValueError(f"{num_experts} experts do not shard evenly over {world} ranks")
    per = num_experts // world
    return rank * per, (rank + 1) * per
