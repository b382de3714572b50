"""Expert-parallel decomposition on CPU: world_size 2 and 4 over ``gloo``.

The product path runs the library's NCCL all-gather / reduce-scatter and the CUDA layer; here
``moe_w4a16_ep`` gets a CPU exchange built from torch.distributed (gloo) and the oracle, so the
dispatch (all-gather of tokens and routing), the per-rank expert localisation, the fp32 partial
combine and the reduce-scatter + single rounding are checked against the single-process oracle
forward on the same inputs."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import moe_oracle as O

T, E, K_TOP, H, I = 6, 8, 3, 128, 128


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class _W:  # the slice of MoEWeights the EP path reads
    def __init__(self, w13, w2):
        self.w13d, self.w2d = w13, w2
        self.num_experts, self.hidden, self.inter = w13.shape[0], w13.shape[2], w2.shape[2]


class CpuExchange:
    """Same contract as ep.NcclExchange, on gloo + the oracle."""

    def __init__(self):
        self.world, self.rank = dist.get_world_size(), dist.get_rank()

    def dispatch(self, x, ids, w):
        out = []
        for t in (x, ids, w):
            parts = [torch.empty_like(t) for _ in range(self.world)]
            dist.all_gather(parts, t)
            out.append(torch.cat(parts))
        return tuple(out)

    @staticmethod
    def localize(ids_all, base, n):
        loc = ids_all - base
        return torch.where((loc >= 0) & (loc < n), loc, torch.full_like(loc, -1))

    @staticmethod
    def experts(x_all, weights, w_all, ids_local, ntok=0, timer=None):
        """Local experts over the node batch; fp32 weighted sums, NOT rounded (the partial)."""
        ids, w = ids_local.numpy(), w_all.numpy()
        counts, offsets, sorted_pairs, pair_pos = O.moe_permute(ids, weights.num_experts)
        xp = x_all.numpy()[sorted_pairs[:offsets[-1]] // ids.shape[1]]
        h = O.grouped_gemm(xp, weights.w13d, counts, offsets, "f16", gated=True)
        yp = O.grouped_gemm(h, weights.w2d, counts, offsets, "f16", gated=False)
        part = np.zeros((ids.shape[0], yp.shape[1]), np.float32)
        for j in range(ids.shape[1]):
            pos = pair_pos.reshape(ids.shape)[:, j]
            ok = pos >= 0
            part[ok] += w[ok, j:j + 1] * yp[pos[ok]]
        return torch.from_numpy(part)

    def combine(self, partial, T_, dtype):
        total = partial.clone()
        dist.all_reduce(total)  # gloo: reduce-scatter = all-reduce + this rank's slice
        mine = total[self.rank * T_:(self.rank + 1) * T_]
        return torch.from_numpy(O.round_act(mine.numpy(), "f16"))


def _inputs(world=2):
    rng = np.random.default_rng(11)
    q13, z13, s13 = O.synth_awq_expert_weights(rng, E, 2 * I, H, "f16")
    q2, z2, s2 = O.synth_awq_expert_weights(rng, E, H, I, "f16")
    w13, w2 = O.dequant(q13, z13, s13, "f16"), O.dequant(q2, z2, s2, "f16")
    xs, ids, wts = [], [], []
    for r in range(world):  # each rank routes its own T tokens
        xs.append(O.round_act(rng.standard_normal((T, H)).astype(np.float32), "f16"))
        lg = rng.standard_normal((T, E)).astype(np.float32)
        i, w = O.route_topk(lg, K_TOP, "softmax", True)
        ids.append(i)
        wts.append(w)
    return w13, w2, xs, ids, wts


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2504_16214_b200.moe.ep import moe_w4a16_ep, shard_bounds
    w13, w2, xs, ids, wts = _inputs(world)
    lo, hi = shard_bounds(E, world, rank)
    y = moe_w4a16_ep(torch.from_numpy(xs[rank]), _W(w13[lo:hi], w2[lo:hi]), torch.from_numpy(wts[rank]),
                     torch.from_numpy(ids[rank]), exchange=CpuExchange())
    q.put((rank, y.numpy()))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_ep_matches_single_process_oracle(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    w13, w2, xs, ids, wts = _inputs(world)
    for r in range(world):
        want = O.moe_forward(xs[r], w13, w2, ids[r], wts[r], "f16")
        # per-rank GEMMs see different row batches (BLAS blocking) and the fp32 sum runs over ranks
        # in a different order -> last-ulp fp16 differences only
        np.testing.assert_allclose(got[r], want, rtol=2e-3, atol=1e-4)


def test_localize_rule():
    """ids outside [base, base + n) are dropped (-1): the CPU rule the CUDA ep_localize kernel follows."""
    ids = torch.tensor([[0, 3, 5], [7, 2, -1]], dtype=torch.int32)
    assert CpuExchange.localize(ids, 2, 4).tolist() == [[-1, 1, 3], [-1, 0, -1]]


def test_shard_with_shared_layout():
    """[routed | shared] packed weights -> (this rank's routed shard, the replicated shared experts)."""
    from paper_2504_16214_b200.moe.ep import shard_with_shared
    from paper_2504_16214_b200.moe.weights import MoEWeights, PackedW4
    per13, per2 = 10, 6
    E, S, world = 8, 1, 4
    full = MoEWeights(PackedW4(torch.arange((E + S) * per13), E + S, 256, 128, 2, torch.float16),
                      PackedW4(torch.arange((E + S) * per2), E + S, 128, 128, 1, torch.float16))
    for rank in range(world):
        routed, shared = shard_with_shared(full, S, world, rank)
        assert routed.num_experts == 2 and shared.num_experts == 1
        assert routed.w13.blocks.tolist() == list(range(2 * rank * per13, (2 * rank + 2) * per13))
        assert shared.w2.blocks.tolist() == list(range(E * per2, (E + S) * per2))


def test_ep_shared_experts_need_explicit_weights():
    from paper_2504_16214_b200.moe import fused_moe_w4a16
    from paper_2504_16214_b200.moe.weights import MoEWeights, PackedW4
    w = MoEWeights(PackedW4(torch.zeros(4), 2, 256, 128, 2, torch.float16),
                   PackedW4(torch.zeros(4), 2, 128, 128, 1, torch.float16))
    with pytest.raises(ValueError, match="shared_weights"):
        fused_moe_w4a16(torch.zeros(2, 128), torch.zeros(2, 1), w, 1, ep_group=object(), num_shared_experts=1)
