"""MoE operator entry points (Python host side).

The reference exposes no MoE operator (``/root/reference/pkg/src/tilesynth/__init__.py:16-58`` is
layout synthesis only). The entry points mirror the call the paper's kernel is
dropped into -- vLLM's ``fused_experts(hidden_states, w1, w2, topk_weights, topk_ids, ...)``
(``vllm/model_executor/layers/fused_moe/fused_moe.py:1587-1597``) -- with AWQ int4 weights packed
once by :mod:`.weights`:

* :func:`moe_w4a16` -- routed experts for precomputed ``topk_weights`` / ``topk_ids``;
* :func:`fused_moe_w4a16` -- router logits in, top-k routing on the device, then :func:`moe_w4a16`;
* :func:`select_experts` -- the routing step alone.

Pipeline (all on the current stream, no host synchronisation): permute -> gather -> gate/up
grouped GEMM with fused SiLU*up -> down grouped GEMM -> weighted combine. With ``ep_group`` set
the experts are sharded across ranks and tokens travel by all-to-all (:mod:`.ep`).
"""
from __future__ import annotations

import contextlib
import os
import threading

import torch

from . import ops
from .weights import MoEWeights, pack_moe_awq


def select_experts(router_logits: torch.Tensor, top_k: int, scoring: str = "softmax",
                   renormalize: bool = False, num_expert_group: int = 0, topk_group: int = 0,
                   e_score_correction_bias: torch.Tensor | None = None, routed_scaling_factor: float = 1.0):
    """-> (topk_weights fp32 [T, k], topk_ids int32 [T, k]); ties go to the lower expert id.
    ``num_expert_group`` > 0 selects DeepSeek-V3/R1 grouped top-k (vLLM ``grouped_topk``: groups,
    ``topk_group`` kept groups, optional correction bias, ``routed_scaling_factor``)."""
    logits = router_logits.float().contiguous()
    if num_expert_group:
        ids, wts = ops.route_grouped_topk(logits, top_k, num_expert_group, topk_group, scoring, renormalize,
                                          e_score_correction_bias, routed_scaling_factor)
    else:
        ids, wts = ops.route_topk(logits, top_k, scoring, renormalize)
        if routed_scaling_factor != 1.0:
            wts = wts * routed_scaling_factor
    return wts, ids


class _Workspace:
    """Grow-only scratch so steady-state calls allocate nothing. Buffers are keyed by (device,
    stream): two layer calls in flight on different streams never share intermediates. A captured
    FusedMoEGraph owns a private instance (see :func:`_use_workspace`), so its replays cannot collide
    with eager calls or with other graphs either."""

    def __init__(self, per_stream: bool = True):
        self.buf: dict[tuple, torch.Tensor] = {}
        self.per_stream = per_stream

    def get(self, name: str, shape, dtype, device) -> torch.Tensor:
        n = 1
        for s in shape:
            n *= s
        dev = torch.device(device)
        key = (name, dtype, str(dev), torch.cuda.current_stream(dev).cuda_stream if self.per_stream else 0)
        t = self.buf.get(key)
        if t is None or t.numel() < n:
            t = torch.empty(max(n, 1), dtype=dtype, device=dev)
            self.buf[key] = t
        return t[:n].view(*shape)


_default_ws = _Workspace()
_active = threading.local()


class _WsProxy:
    """The workspace of the current thread: a graph's private one while it is warmed up / captured,
    else the process default (keyed by stream)."""

    def get(self, *a):
        return (getattr(_active, "ws", None) or _default_ws).get(*a)


_ws = _WsProxy()


@contextlib.contextmanager
def _use_workspace(ws: _Workspace):
    prev = getattr(_active, "ws", None)
    _active.ws = ws
    try:
        yield ws
    finally:
        _active.ws = prev


# fused route + permute (one CTA) up to this many (token, slot) pairs; 0 disables. Measured: ~1 us faster
# for DS-R1 T=1 (8 pairs), a wash at T=16 and slower from T=64 on (one CTA routes every token, where
# the separate routing kernel spreads tokens over SMs), so only the smallest batches use it.
_ROUTE_PERMUTE_MAX_PAIRS = int(os.environ.get("W4A16_ROUTE_PERMUTE_MAX_PAIRS", "64"))
# experiment (W4A16_FUSED_GATHER=1): the gate/up GEMM gathers x's rows itself (TMA gather4 in its
# producer) instead of a gather kernel. Correct (bit-identical) but measured 1.5x slower at T=64 and 2.8x
# slower gate/up at T=8192: 64 four-row gather4 requests per 49 KB stage throttle the TMA unit.
_FUSED_GATHER = os.environ.get("W4A16_FUSED_GATHER", "0") not in ("", "0")
# decode: h's group sums from the gate/up epilogue instead of a separate kernel -- W4A16_FUSED_OSUM=1 / 0
# forces it on / off; unset: by rows per expert (see moe_w4a16)
_FUSED_OSUM = None if os.environ.get("W4A16_FUSED_OSUM", "") == "" else os.environ["W4A16_FUSED_OSUM"] != "0"
# largest token tile that runs the offset-code (decode) GEMM; larger tiles dequantise with the scale


class KernelTimer:
    """Optional per-kernel CUDA-event recorder (used by bench.py to time the dominant kernel live
    on the launching stream). ``timer.mark(name)`` brackets the next launch."""

    def __init__(self):
        self.events: dict[str, list] = {}

    def span(self, name: str):
        timer = self

        class _Span:
            def __enter__(self):
                self.a = torch.cuda.Event(enable_timing=True)
                self.b = torch.cuda.Event(enable_timing=True)
                self.a.record()

            def __exit__(self, *exc):
                self.b.record()
                timer.events.setdefault(name, []).append((self.a, self.b))

        return _Span()

    def mean_ms(self, name: str) -> float:
        ev = self.events.get(name, [])
        return sum(a.elapsed_time(b) for a, b in ev) / max(1, len(ev))

    def count(self) -> int:
        return sum(len(v) for v in self.events.values())


class _NoTimer:
    class _Null:
        def __enter__(self):
            return None

        def __exit__(self, *exc):
            return False

    _null = _Null()

    def span(self, name):
        return self._null


_NOTIMER = _NoTimer()


_AWQ_CACHE: dict = {}


def _packed_from_awq(w13_q, w13_s, w13_z, w2_q, w2_s, w2_z, group_size):
    """Raw AWQ tensors -> MoEWeights, repacked once per (tensor storage, version) and cached (the
    vLLM process_weights_after_loading step, done lazily)."""
    key = tuple((t.data_ptr(), t._version, tuple(t.shape)) for t in (w13_q, w13_s, w13_z, w2_q, w2_s, w2_z))
    hit = _AWQ_CACHE.get(key)
    if hit is None:
        if len(_AWQ_CACHE) > 64:
            _AWQ_CACHE.clear()
        hit = _AWQ_CACHE[key] = pack_moe_awq(w13_q, w13_s, w13_z, w2_q, w2_s, w2_z, group_size)
    return hit


def moe_w4a16(x: torch.Tensor, weights, topk_weights: torch.Tensor, topk_ids: torch.Tensor = None, *awq_rest,
              ep_group=None, ntok: int = 0, timer: KernelTimer | None = None, perm=None, f32_out: bool = False,
              group_size: int = 128) -> torch.Tensor:
    """y[t] = sum_j topk_weights[t, j] * Expert_{topk_ids[t, j]}(x[t]) for the W4A16 SwiGLU experts.

    ``x`` [T, H] fp16/bf16 on CUDA; ``topk_ids`` int32 [T, k]; ``topk_weights`` fp32 [T, k].
    ``weights`` is a :class:`MoEWeights` -- or, the raw-AWQ form of SURVEY.md 8(b),
    ``moe_w4a16(x, w13_q, w13_s, w13_z, w2_q, w2_s, w2_z, topk_weights, topk_ids, group_size=128,
    ep_group=None)`` with vLLM's AWQ MoE tensors (qweight [E, K, N/8] int32, scales [E, K/G, N],
    qzeros [E, K/G, N/8] int32), repacked on first use. ``f32_out``: return the fp32 sums unrounded
    (the expert-parallel partial)."""
    if isinstance(weights, torch.Tensor):
        if len(awq_rest) != 5:
            raise TypeError("moe_w4a16(x, w13_q, w13_s, w13_z, w2_q, w2_s, w2_z, topk_weights, topk_ids, ...)")
        w2_q, w2_s, w2_z, topk_weights_, topk_ids_ = awq_rest
        weights = _packed_from_awq(weights, topk_weights, topk_ids, w2_q, w2_s, w2_z, group_size)
        topk_weights, topk_ids = topk_weights_, topk_ids_
    elif awq_rest or topk_ids is None:
        raise TypeError("moe_w4a16(x, weights, topk_weights, topk_ids, ...)")
    if ep_group is not None:
        from .ep import moe_w4a16_ep
        return moe_w4a16_ep(x, weights, topk_weights, topk_ids, ep_group, ntok=ntok, timer=timer)
    tm = timer or _NOTIMER
    T, H = x.shape
    if T == 0:  # empty batch (single GPU): nothing to launch
        return x.new_empty((0, H), dtype=torch.float32 if f32_out else x.dtype)
    if H != weights.hidden:
        raise ValueError(f"hidden size {H} != packed weights' {weights.hidden}")
    if x.dtype != weights.w13.dtype:
        raise ValueError(f"activation dtype {x.dtype} != weight scale dtype {weights.w13.dtype}")
    x = x.contiguous()
    topk_ids = topk_ids.to(torch.int32).contiguous()
    topk_weights = topk_weights.to(torch.float32).contiguous()
    k = topk_ids.shape[1]
    E, I = weights.num_experts, weights.inter
    P = T * k
    dev = x.device
    if perm is not None:  # (counts, offsets, sorted_pairs, pair_pos) already computed with the routing
        counts, offsets, sorted_pairs, pair_pos = perm
    else:
        with tm.span("permute"):
            counts, offsets, sorted_pairs, pair_pos = ops.moe_permute(
                topk_ids, E, _ws.get("perm_ws", (max(ops.permute_ws_bytes(P, E), 1),), torch.uint8, dev))
    nt = ntok or ops.pick_ntok(P, E)
    decode = nt <= ops.decode_max_ntok()  # offset-code GEMMs: per-group activation sums ride along with X and h
    if _FUSED_GATHER:  # the gate/up producer gathers x's rows itself (TMA gather4); decode sums over x
        xp = None
        if decode:
            with tm.span("sums_x"):
                xs = ops.group_sums(x, out=_ws.get("xs", ops.sums_shape(T, H), torch.float32, dev))
        else:
            xs = None
    else:
        with tm.span("gather"):
            xp_buf = _ws.get("xp", (P, H), x.dtype, dev)
            if decode:
                xp, xs = ops.moe_gather_sums(x, sorted_pairs, k, P, offsets[E:], out=xp_buf,
                                             sums=_ws.get("xs", ops.sums_shape(P, H), torch.float32, dev))
            else:
                xp, xs = ops.moe_gather(x, sorted_pairs, k, P, offsets[E:], out=xp_buf), None
    def splitk_ws(K: int, n_out: int, gated: bool):
        # one buffer per GEMM: a captured graph keeps _ws's buffers alive, so neither may be reallocated
        b = ops.gemm_ws_bytes(P, K, E, n_out, gated, nt) if decode else 0
        return _ws.get("splitk_gu" if gated else "splitk_dn", (b,), torch.uint8, dev) if b else None

    hs = _ws.get("hs", ops.sums_shape(P, I), torch.float32, dev) if decode else None
    gu_ws = splitk_ws(H, I, True)
    # h's group sums (the down GEMM's xsum) from the gate/up epilogue: measured ~1 % faster than the
    # separate kernel at <= 2 rows per expert (DS-R1 T <= 64), 3 % slower at 8 (T = 256; the epilogue's
    # per-tile cross-warp reduction grows with the tile's rows)
    want_fused = P <= 4 * E if _FUSED_OSUM is None else _FUSED_OSUM
    fused_osum = decode and want_fused  # (with split-K the C entry point runs the sums pass itself)
    with tm.span("gemm_gate_up"):
        h_buf = _ws.get("h", (P, I), x.dtype, dev)
        if xp is None:
            h = ops.grouped_gemm_gather(x, sorted_pairs, k, weights.w13.blocks, E, I, True, counts, offsets, nt,
                                        out=h_buf, xsum=xs, workspace=gu_ws, osum=hs if fused_osum else None, rows=P)
        else:
            h = ops.grouped_gemm(xp, weights.w13.blocks, E, I, True, counts, offsets, nt, out=h_buf, xsum=xs,
                                 workspace=gu_ws, osum=hs if fused_osum else None)
    if decode and not fused_osum:
        with tm.span("sums_h"):
            ops.group_sums(h, offsets[E:], out=hs)
    with tm.span("gemm_down"):
        yp = ops.grouped_gemm(h, weights.w2.blocks, E, H, False, counts, offsets, nt,
                              out=_ws.get("yp", (P, H), x.dtype, dev), xsum=hs, workspace=splitk_ws(I, H, False))
    with tm.span("combine"):
        return ops.moe_combine(yp, pair_pos, topk_weights, f32=f32_out)


def with_shared_experts(topk_weights: torch.Tensor, topk_ids: torch.Tensor, first_shared: int, num_shared: int,
                        scale: float = 1.0):
    """Append the always-active shared experts (DeepSeek-V3/R1: one) as extra routing slots of weight
    ``scale``: the grouped GEMMs then run them next to the routed experts, and the combine adds their
    output -- y = sum_j w_j E_{id_j}(x) + scale * sum_s Shared_s(x). Shared expert s is expert
    ``first_shared + s`` of the packed weights."""
    T = topk_ids.shape[0]
    sid = torch.arange(first_shared, first_shared + num_shared, dtype=torch.int32, device=topk_ids.device)
    ids = torch.cat([topk_ids.to(torch.int32), sid.expand(T, num_shared)], dim=1).contiguous()
    wts = torch.cat([topk_weights.float(), topk_weights.new_full((T, num_shared), scale, dtype=torch.float32)],
                    dim=1).contiguous()
    return wts, ids


def fused_moe_w4a16(x: torch.Tensor, router_logits: torch.Tensor, weights: MoEWeights, top_k: int,
                    scoring: str = "softmax", renormalize: bool = False, ep_group=None,
                    timer: KernelTimer | None = None, num_expert_group: int = 0, topk_group: int = 0,
                    e_score_correction_bias: torch.Tensor | None = None,
                    routed_scaling_factor: float = 1.0, num_shared_experts: int = 0,
                    shared_weights: MoEWeights | None = None) -> torch.Tensor:
    """Shared experts (always active, weight 1; the router logits cover only the routed experts):

    * ``shared_weights`` given: they are those experts (``num_shared_experts`` defaults to their
      count) and ``weights`` holds only routed experts -- the full set on one GPU, this rank's
      contiguous shard (:func:`~.ep.shard_bounds`) under ``ep_group``;
    * else ``num_shared_experts`` > 0 on one GPU: the last experts of ``weights`` are the shared ones.
      Under ``ep_group`` this needs ``shared_weights`` (a routed shard plus a shared tail cannot be
      told apart from a larger shard; :func:`~.ep.shard_with_shared` builds both pieces)."""
    if shared_weights is not None:
        num_shared_experts = num_shared_experts or shared_weights.num_experts
        if num_shared_experts != shared_weights.num_experts:
            raise ValueError(f"num_shared_experts={num_shared_experts} but shared_weights holds "
                             f"{shared_weights.num_experts}")
    elif num_shared_experts and ep_group is not None:
        raise ValueError("expert parallel with shared experts: pass shared_weights= (see ep.shard_with_shared)")
    T = router_logits.shape[0]
    if T == 0 and ep_group is None:  # (EP ranks with no tokens still join the exchanges)
        return x.new_empty((0, x.shape[1]))
    if (ep_group is None and not num_expert_group and not num_shared_experts and routed_scaling_factor == 1.0
            and T * top_k <= _ROUTE_PERMUTE_MAX_PAIRS):
        # small batch: routing and the permutation in one single-CTA kernel
        with (timer or _NOTIMER).span("route_permute"):
            ids, wts, counts, offsets, sp, pp = ops.route_permute(router_logits.float().contiguous(), top_k, scoring,
                                                                  renormalize)
        return moe_w4a16(x, weights, wts, ids, timer=timer, perm=(counts, offsets, sp, pp))
    with (timer or _NOTIMER).span("route"):
        topk_weights, topk_ids = select_experts(router_logits, top_k, scoring, renormalize, num_expert_group,
                                                topk_group, e_score_correction_bias, routed_scaling_factor)
    if not num_shared_experts:
        return moe_w4a16(x, weights, topk_weights, topk_ids, ep_group=ep_group, timer=timer)
    if ep_group is not None:
        # expert parallel: the routed shard goes through the exchange, the (replicated) shared experts
        # run data-parallel on this rank's own tokens
        y = moe_w4a16(x, weights, topk_weights, topk_ids, ep_group=ep_group, timer=timer)
        if not x.shape[0]:
            return y
        sw, sid = with_shared_experts(topk_weights[:, :0], topk_ids[:, :0], 0, num_shared_experts)
        return y.add_(moe_w4a16(x, shared_weights, sw, sid, timer=timer))
    if shared_weights is not None:  # one GPU: run routed + shared in the same grouped GEMMs
        weights = concat_experts(weights, shared_weights)
    first = weights.num_experts - num_shared_experts
    topk_weights, topk_ids = with_shared_experts(topk_weights, topk_ids, first, num_shared_experts)
    return moe_w4a16(x, weights, topk_weights, topk_ids, timer=timer)


_CONCAT_CACHE: dict = {}


def concat_experts(a: MoEWeights, b: MoEWeights) -> MoEWeights:
    """[a's experts | b's experts] as one MoEWeights (one copy, cached per (a, b) buffer pair)."""
    key = (a.w13.blocks.data_ptr(), a.w2.blocks.data_ptr(), b.w13.blocks.data_ptr(), b.w2.blocks.data_ptr(),
           a.num_experts, b.num_experts)
    hit = _CONCAT_CACHE.get(key)
    if hit is None:
        hit = a.concat(b)
        _CONCAT_CACHE[key] = hit
    return hit


class FusedMoEGraph:
    """The single-GPU layer (routing -> permute -> gather -> gate/up -> down -> combine) captured once
    into a CUDA graph for fixed (tokens, dtype) and replayed per call -- the decode-serving mode, where
    the step is otherwise bound by host launch overhead (7 launches). Inputs are copied into the
    graph's own buffers; the returned output tensor is the graph's (overwritten by the next call)."""

    def __init__(self, weights: MoEWeights, tokens: int, top_k: int, scoring: str = "softmax",
                 renormalize: bool = False, dtype: torch.dtype = torch.float16, device=None,
                 x: torch.Tensor | None = None, router_logits: torch.Tensor | None = None,
                 num_shared_experts: int = 0, workspace: _Workspace | None = None, ep_group=None,
                 shared_weights: MoEWeights | None = None):
        """``workspace``: the graph's private intermediates (default: its own). Graphs that share one
        must be replayed in stream order (FusedMoEPipeline's two slots do). ``ep_group``: capture the
        expert-parallel layer (its NCCL all-gather / reduce-scatter are captured too; ``weights`` is
        this rank's shard, the router logits cover all experts of the group)."""
        dev = torch.device(device) if device is not None else weights.w13.blocks.device
        self.workspace = workspace or _Workspace(per_stream=False)
        self.x = torch.zeros((tokens, weights.hidden), dtype=dtype, device=dev)
        import torch.distributed as dist
        n_routed = (weights.num_experts * (dist.get_world_size(ep_group) if ep_group is not None else 1)
                    - (num_shared_experts if shared_weights is None else 0))
        self.logits = torch.randn((tokens, n_routed), device=dev)
        if x is not None:  # warm up / capture on the caller's first inputs (same routing as served)
            self.x.copy_(x)
        if router_logits is not None:
            self.logits.copy_(router_logits)
        args = (weights, top_k, scoring, renormalize)
        kw = {"num_shared_experts": num_shared_experts, "ep_group": ep_group, "shared_weights": shared_weights}
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with _use_workspace(self.workspace):
            with torch.cuda.stream(side):  # warm-up: kernel attributes, workspace growth, first launches
                for _ in range(2):
                    fused_moe_w4a16(self.x, self.logits, *args, **kw)
            torch.cuda.current_stream(dev).wait_stream(side)
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph):
                self.y = fused_moe_w4a16(self.x, self.logits, *args, **kw)

    def __call__(self, x: torch.Tensor | None = None, router_logits: torch.Tensor | None = None) -> torch.Tensor:
        if x is not None:
            self.x.copy_(x, non_blocking=True)
        if router_logits is not None:
            self.logits.copy_(router_logits, non_blocking=True)
        self.graph.replay()
        return self.y


class FusedMoEPipeline:
    """Serving loop over host batches with the copies off the critical path: the host->device copy
    of step i+1 and the device->host copy of step i run on their own streams while step i's layer
    (a FusedMoEGraph replay) runs. Two graph slots (own input and output buffers; weights and
    workspaces shared, replays serialised on the caller's stream) make that safe:

        pipe = FusedMoEPipeline(weights, tokens, top_k, ...)
        pipe.start()
        for x_h, lg_h, y_h in batches:   # pinned host tensors
            pipe(x_h, lg_h, y_h)         # enqueue only: H2D, layer, D2H
        pipe.finish()                    # the caller's stream now waits for the last D2H

    Every step still moves its own inputs in and its own output out; only the overlap changes."""

    def __init__(self, weights: MoEWeights, tokens: int, top_k: int, scoring: str = "softmax",
                 renormalize: bool = False, dtype: torch.dtype = torch.float16, device=None,
                 x: torch.Tensor | None = None, router_logits: torch.Tensor | None = None, ep_group=None):
        self.dev = torch.device(device) if device is not None else weights.w13.blocks.device
        ws = _Workspace(per_stream=False)  # shared by both slots: their replays are serialised on one stream
        self.slots = [FusedMoEGraph(weights, tokens, top_k, scoring, renormalize, dtype, self.dev, x, router_logits,
                                    workspace=ws, ep_group=ep_group) for _ in range(2)]
        self.h2d = torch.cuda.Stream(device=self.dev)
        self.d2h = torch.cuda.Stream(device=self.dev)
        self.i = 0
        self._reset_events()

    def _reset_events(self):
        mk = lambda: [torch.cuda.Event(), torch.cuda.Event()]  # noqa: E731
        self.h2d_done, self.comp_done, self.d2h_done = mk(), mk(), mk()
        self.used = [False, False]

    def start(self):
        """Order the copy streams after everything already queued on the caller's stream."""
        cur = torch.cuda.current_stream(self.dev)
        self.h2d.wait_stream(cur)
        self.d2h.wait_stream(cur)

    def __call__(self, x_host: torch.Tensor, logits_host: torch.Tensor, y_host: torch.Tensor) -> torch.Tensor:
        s = self.i & 1
        self.i += 1
        g = self.slots[s]
        cur = torch.cuda.current_stream(self.dev)
        if self.used[s]:  # the slot's inputs are free once its previous replay is done
            self.h2d.wait_event(self.comp_done[s])
        with torch.cuda.stream(self.h2d):
            g.x.copy_(x_host, non_blocking=True)
            g.logits.copy_(logits_host, non_blocking=True)
            self.h2d_done[s].record(self.h2d)
        cur.wait_event(self.h2d_done[s])
        if self.used[s]:  # and its output once the previous device->host copy is done
            cur.wait_event(self.d2h_done[s])
        g.graph.replay()
        self.comp_done[s].record(cur)
        self.d2h.wait_event(self.comp_done[s])
        with torch.cuda.stream(self.d2h):
            y_host.copy_(g.y, non_blocking=True)
            self.d2h_done[s].record(self.d2h)
        self.used[s] = True
        return y_host

    def finish(self):
        """The caller's stream waits for every queued copy (y_host of every step is then valid once
        that stream reaches this point)."""
        cur = torch.cuda.current_stream(self.dev)
        cur.wait_stream(self.d2h)
        cur.wait_stream(self.h2d)


_LINEAR_ROUTING: dict = {}


def w4a16_linear(x: torch.Tensor, w, ntok: int = 0) -> torch.Tensor:
    """Dense W4A16 linear y = x @ W^T (one "expert"; BASELINE config 2). ``w`` is a PackedW4 with
    num_experts == 1 and parts == 1."""
    M, K = x.shape
    dev = x.device
    key = (M, str(dev))
    if key not in _LINEAR_ROUTING:  # cached: no host->device copy per call (CUDA-graph capturable)
        _LINEAR_ROUTING[key] = (torch.tensor([M], dtype=torch.int32, device=dev),
                                torch.tensor([0, M], dtype=torch.int32, device=dev))
    counts, offsets = _LINEAR_ROUTING[key]
    nt = ntok or ops.pick_ntok(M, 1)
    x = x.contiguous()
    decode = nt <= ops.decode_max_ntok()
    xs = ops.group_sums(x) if decode else None
    wsb = ops.gemm_ws_bytes(M, K, 1, w.n_rows, False, nt) if decode else 0
    ws = _ws.get("linear_splitk", (wsb,), torch.uint8, dev) if wsb else None
    return ops.grouped_gemm(x, w.blocks, 1, w.n_rows, False, counts, offsets, nt, xsum=xs, workspace=ws)
