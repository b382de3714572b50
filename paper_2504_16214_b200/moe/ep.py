"""Expert parallelism: experts sharded contiguously across the ranks of one node; tokens reach them
by an all-gather and come back by a reduce-scatter, both NCCL collectives over NVLink / NVSwitch run
by this library (``csrc/moe_ep.cu``, C ABI ``w4a16_ep_*``) on its own communicator.

Rank r owns global experts [r*E_l, (r+1)*E_l). With T tokens on every rank:

  1. dispatch: all-gather x [T, H], topk_ids and topk_weights [T, k] -> the node batch [world*T];
  2. localize: ids outside this rank's shard become -1 (the permutation drops them);
  3. the single-GPU layer (permute -> gather -> gate/up -> down -> combine) on the local pairs, with
     the combine's fp32 sums left unrounded: this rank's partial output for every node token;
  4. combine: reduce-scatter the fp32 partials (sum over ranks) and round once -> [T, H].

Every shape is fixed by (world, T, k, H), so nothing is read back to the host and the whole step can
be captured in a CUDA graph (the all-to-all(v) alternative needs its split sizes on the host). The
traffic per rank -- world*T*H activations in, world*T*H fp32 out -- matches an all-to-all of the
T*k routed rows when k = world (DS-R1 top-8 on 8 GPUs), and NCCL runs both collectives with in-switch
multicast / reduction (NVLS) on NVSwitch systems. Every rank must pass the same T.

``exchange`` supplies the collectives and the local layer; the product path is :class:`NcclExchange`,
the tests inject a CPU exchange over ``gloo`` (world size 2 and 4) to check the decomposition.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import ops


class EPComm:
    """This library's NCCL communicator for one torch.distributed group (created once per group,
    collectively: the group's first rank makes the unique id, the group broadcasts it)."""

    _by_group: dict = {}

    def __init__(self, group=None):
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        uid = [ops.ep_unique_id() if self.rank == 0 else None]
        src = dist.get_global_rank(group, 0) if group is not None else 0
        dist.broadcast_object_list(uid, src=src, group=group)
        self.handle = ops.ep_comm_init(uid[0], self.rank, self.world)

    @classmethod
    def of(cls, group=None) -> "EPComm":
        """The communicator of ``group`` (None = the default group), created on first use. Keyed by
        the group object itself, which the cache keeps alive, so a new group never aliases an old
        one's entry."""
        if group not in cls._by_group:
            cls._by_group[group] = cls(group)
        return cls._by_group[group]


class NcclExchange:
    """Product path: all-gather / reduce-scatter through the library's NCCL communicator."""

    def __init__(self, group=None):
        self.comm = EPComm.of(group)
        self.world, self.rank = self.comm.world, self.comm.rank

    def dispatch(self, x, topk_ids, topk_weights):
        return ops.ep_dispatch(self.comm.handle, self.world, x, topk_ids, topk_weights)

    @staticmethod
    def localize(ids_all, base, local_experts):
        return ops.ep_localize(ids_all, base, local_experts)

    def experts(self, x_all, weights, w_all, ids_local, ntok=0, timer=None):
        """The local layer over the node batch; the token tile is sized for the pairs expected on
        this rank (1/world of them under uniform routing -- the rest are other ranks' ids, -1)."""
        from .layer import moe_w4a16
        nt = ntok or ops.pick_ntok(ids_local.numel() // self.world, weights.num_experts)
        return moe_w4a16(x_all, weights, w_all, ids_local, ntok=nt, timer=timer, f32_out=True)

    def combine(self, partial, T, dtype):
        return ops.ep_combine(self.comm.handle, partial, T, dtype)


def moe_w4a16_ep(x: torch.Tensor, weights, topk_weights: torch.Tensor, topk_ids: torch.Tensor, group=None,
                 ntok: int = 0, timer=None, exchange=None) -> torch.Tensor:
    """Expert-parallel W4A16 MoE. ``weights`` holds this rank's contiguous expert shard;
    ``topk_ids`` are global expert ids; every rank passes the same number of tokens."""
    from .layer import _NOTIMER
    tm = timer or _NOTIMER
    ex = exchange or NcclExchange(group)
    T = x.shape[0]
    if T == 0:
        return x.new_empty((0, x.shape[1]))
    e_local = weights.num_experts
    with tm.span("dispatch"):
        x_all, ids_all, w_all = ex.dispatch(x.contiguous(), topk_ids.to(torch.int32).contiguous(),
                                            topk_weights.to(torch.float32).contiguous())
    with tm.span("localize"):
        ids_local = ex.localize(ids_all, ex.rank * e_local, e_local)
    partial = ex.experts(x_all, weights, w_all, ids_local, ntok, timer)
    with tm.span("ep_combine"):
        return ex.combine(partial, T, x.dtype)


def local_expert_ids(recv_counts: torch.Tensor, n_recv: int | None = None) -> torch.Tensor:
    """Local expert id of every row an all-to-all delivered grouped by (source rank, local expert)
    with counts ``recv_counts`` [world, E_l] -- the rule the C entry ``w4a16_ep_local_order`` (kept
    for all-to-all based callers) orders by."""
    world, e_local = recv_counts.shape
    experts = torch.arange(e_local, device=recv_counts.device, dtype=torch.int32).repeat(world)
    return torch.repeat_interleave(experts, recv_counts.reshape(-1).to(torch.int64),
                                   output_size=n_recv).to(torch.int32)


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
