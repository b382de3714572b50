"""Expert-parallel exchange plumbing on CPU: world_size 2 and 4 over ``gloo``.

The product path runs the CUDA ops; here ``moe_w4a16_ep`` gets a CPU backend built from the oracle
so the dispatch plan, the two all-to-alls, the receiver-side local-expert permutation and the
combine are checked against the single-process oracle forward on the same inputs."""
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


class CpuBackend:
    @staticmethod
    def permute(ids, n_exp):
        c, o, sp, pp = O.moe_permute(ids.numpy(), n_exp)
        return (torch.from_numpy(c), torch.from_numpy(o), torch.from_numpy(sp), torch.from_numpy(pp))

    @staticmethod
    def gather(x, sorted_pairs, topk, rows, row_limit=None):
        if row_limit is not None:
            rows = min(rows, int(row_limit[0]))
        idx = sorted_pairs[:rows].long() // topk
        return x[idx].clone()

    @staticmethod
    def combine(y_back, pair_pos, w):
        Tn, k = w.shape
        y = torch.zeros((Tn, y_back.shape[1]), dtype=torch.float32)
        pp = pair_pos.view(Tn, k)
        for j in range(k):
            ok = pp[:, j] >= 0
            y[ok] += w[ok, j:j + 1] * y_back[pp[ok, j].long()]
        return torch.from_numpy(O.round_act(y.numpy(), "f16"))

    @staticmethod
    def experts(x, weights, counts, offsets, ntok, timer=None):
        h = O.grouped_gemm(x.numpy(), weights.w13d, counts.numpy(), offsets.numpy(), "f16", gated=True)
        y = O.grouped_gemm(h, weights.w2d, counts.numpy(), offsets.numpy(), "f16", gated=False)
        return torch.from_numpy(y)


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
                     torch.from_numpy(ids[rank]), backend=CpuBackend)
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
        # per-rank GEMMs see different row batches (BLAS blocking) -> last-ulp fp16 differences only
        np.testing.assert_allclose(got[r], want, rtol=2e-3, atol=1e-4)


def test_local_expert_ids_and_plan_shapes():
    from paper_2504_16214_b200.moe.ep import local_expert_ids
    rc = torch.tensor([[2, 0, 1], [0, 3, 1]], dtype=torch.int32)
    assert local_expert_ids(rc).tolist() == [0, 0, 2, 1, 1, 1, 2]


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
