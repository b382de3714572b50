"""GPU parity tests: every CUDA kernel of the W4A16 MoE path against the CPU oracle
(``oracle/moe_oracle.py``), called through the C ABI (ctypes) via the host wrappers.

Bars (north star): bit-exact for dequantised weights, routing ids and permutation indices;
rtol 1e-2 / atol 1e-2 for GEMM / layer outputs (fp32 accumulate)."""
import numpy as np
import pytest
import torch

import moe_oracle as O

pytestmark = pytest.mark.gpu

RTOL = 1e-2
ATOL = 1e-2
TDT = {"f16": torch.float16, "bf16": torch.bfloat16}


def _ops():
    from paper_2504_16214_b200.moe import ops
    return ops


def _to_dev_act(a: np.ndarray, dt: str) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(O.act_bits(a, dt))).view(TDT[dt]).cuda()


def _from_dev_act(t: torch.Tensor, dt: str) -> np.ndarray:
    return O.bits_to_f32(t.view(torch.int16).cpu().numpy().view(np.uint16), dt)


def _packed(q, z, s, dt, gated):
    from paper_2504_16214_b200.moe.weights import pack_awq
    qw, sc, qz = O.to_awq(q, z, s)
    return pack_awq(torch.from_numpy(qw).cuda(), _to_dev_act(sc, dt), torch.from_numpy(qz).cuda(), gated=gated)


# ------------------------------------------------------------------------------------------- dequant
@pytest.mark.parametrize("dt", ["f16", "bf16"])
@pytest.mark.parametrize("gated", [False, True])
def test_repack_dequant_bit_exact(dt, gated):
    rng = np.random.default_rng(1)
    E, N, K = 3, 256, 384
    q, z, s = O.synth_awq_expert_weights(rng, E, N, K, dt)
    s[0, 0, 0] = O.round_act(np.array([-0.75], np.float32), dt)[0]  # a negative scale and extreme codes too
    q[0, 0, :8] = [0, 15, 0, 15, 7, 8, 15, 0]
    w = _packed(q, z, s, dt, gated)
    got = w.dense()
    torch.cuda.synchronize()
    want = O.dequant(q, z, s, dt)
    got_bits = got.view(torch.int16).cpu().numpy().view(np.uint16)
    want_bits = O.act_bits(want, dt)
    assert got_bits.shape == want_bits.shape
    assert np.array_equal(got_bits, want_bits)


# ------------------------------------------------------------------------------------------- routing
@pytest.mark.parametrize("scoring", ["softmax", "sigmoid"])
@pytest.mark.parametrize("renorm", [False, True])
@pytest.mark.parametrize("E,k", [(8, 2), (64, 6), (256, 8), (128, 8), (1000, 3)])
def test_route_topk(scoring, renorm, E, k):
    rng = np.random.default_rng(E * 7 + k)
    T = 67
    lg = rng.standard_normal((T, E)).astype(np.float32)
    lg[3, :] = 0.25                                  # all tied -> ids 0..k-1
    lg[5, E // 2] = lg[5, E // 3] = lg[5].max() + 1  # tie at the top
    lg[7, 1::2] = -np.inf                            # masked experts (half the row)
    lg[8, :] = -np.inf                               # fully masked row: ties -> ids 0..k-1 ...
    lg[8, :k] = 0.0                                  # ... except k finite ones
    ids, w = _ops().route_topk(torch.from_numpy(lg).cuda(), k, scoring, renorm)
    rid, rw = O.route_topk(lg, k, scoring, renorm)
    assert np.array_equal(ids.cpu().numpy(), rid)
    np.testing.assert_allclose(w.cpu().numpy(), rw, rtol=1e-5, atol=1e-6)


@pytest.mark.parametrize("case", [(64, 256, 8, 8, 4, "sigmoid", True, True, 2.5),   # DeepSeek-R1
                                  (33, 256, 8, 8, 4, "sigmoid", True, False, 1.0),
                                  (16, 64, 6, 4, 2, "softmax", False, False, 1.0),
                                  (200, 128, 4, 8, 3, "softmax", True, True, 1.0),
                                  (5, 1024, 8, 32, 6, "sigmoid", True, True, 1.0),
                                  (7, 60, 3, 3, 2, "sigmoid", False, True, 1.0)])
def test_route_grouped_topk(case):
    """DeepSeek-V3/R1 grouped top-k kernel == the oracle (which tests/test_oracle.py pins to vLLM)."""
    T, E, k, G, TG, scoring, renorm, use_bias, scale = case
    rng = np.random.default_rng(T * E + k)
    lg = rng.standard_normal((T, E)).astype(np.float32)
    bias = (rng.standard_normal(E) * 0.1).astype(np.float32) if use_bias else None
    ids, w = _ops().route_grouped_topk(torch.from_numpy(lg).cuda(), k, G, TG, scoring, renorm,
                                       torch.from_numpy(bias).cuda() if bias is not None else None, scale)
    rid, rw = O.grouped_topk(lg, k, G, TG, scoring, renorm, bias, scale)
    assert np.array_equal(ids.cpu().numpy(), rid)
    np.testing.assert_allclose(w.cpu().numpy(), rw, rtol=1e-5, atol=1e-6)


def test_fused_moe_grouped_routing_layer():
    """The layer with DeepSeek-style routing (grouped top-k + bias + scaling) == oracle layer."""
    from paper_2504_16214_b200.moe import fused_moe_w4a16
    from paper_2504_16214_b200.moe.weights import MoEWeights
    rng = np.random.default_rng(5)
    T, E, k, H, I, dt = 24, 32, 4, 256, 256, "f16"
    q13, z13, s13 = O.synth_awq_expert_weights(rng, E, 2 * I, H, dt)
    q2, z2, s2 = O.synth_awq_expert_weights(rng, E, H, I, dt)
    w = MoEWeights(_packed(q13, z13, s13, dt, True), _packed(q2, z2, s2, dt, False))
    x = O.round_act(rng.standard_normal((T, H)).astype(np.float32) * 0.5, dt)
    lg = rng.standard_normal((T, E)).astype(np.float32)
    bias = (rng.standard_normal(E) * 0.1).astype(np.float32)
    y = fused_moe_w4a16(_to_dev_act(x, dt), torch.from_numpy(lg).cuda(), w, k, "sigmoid", True,
                        num_expert_group=4, topk_group=2, e_score_correction_bias=torch.from_numpy(bias).cuda(),
                        routed_scaling_factor=2.5)
    torch.cuda.synchronize()
    rid, rw = O.grouped_topk(lg, k, 4, 2, "sigmoid", True, bias, 2.5)
    want = O.moe_forward(x, O.dequant(q13, z13, s13, dt), O.dequant(q2, z2, s2, dt), rid, rw, dt)
    np.testing.assert_allclose(_from_dev_act(y, dt), want, rtol=RTOL, atol=ATOL)


@pytest.mark.parametrize("T,E,k,scoring", [(1, 256, 8, "softmax"), (64, 256, 8, "softmax"), (37, 128, 8, "sigmoid"),
                                           (200, 8, 2, "softmax"), (512, 256, 8, "softmax"), (3, 1024, 4, "sigmoid")])
def test_route_permute_fused(T, E, k, scoring):
    """Routing + permutation in one CTA == route_topk then moe_permute, bit for bit."""
    ops = _ops()
    rng = np.random.default_rng(T * 3 + E)
    lg = torch.from_numpy(rng.standard_normal((T, E)).astype(np.float32)).cuda()
    ids, w, c, o, sp, pp = ops.route_permute(lg, k, scoring, True)
    ids2, w2 = ops.route_topk(lg, k, scoring, True)
    c2, o2, sp2, pp2 = ops.moe_permute(ids2, E)
    torch.cuda.synchronize()
    assert torch.equal(ids, ids2) and torch.equal(w, w2)
    assert torch.equal(c, c2) and torch.equal(o, o2) and torch.equal(sp, sp2) and torch.equal(pp, pp2)


# ------------------------------------------------------------------------------------------- permute
@pytest.mark.parametrize("P,E", [(1, 4), (64 * 8, 256), (3000, 256), (5000, 7), (65536, 256), (2048, 1024),
                                 (20000, 1024), (9001, 3), (131072, 128)])
def test_permute_bit_exact(P, E):
    rng = np.random.default_rng(P + E)
    ids = rng.integers(0, E, size=P).astype(np.int32)
    if P > 10:
        ids[::11] = -1        # dropped pairs (non-local experts)
        ids[5::13] = E + 3    # out of range -> dropped
    c, o, sp, pp = _ops().moe_permute(torch.from_numpy(ids).cuda(), E)
    rc, ro, rsp, rpp = O.moe_permute(ids, E)
    assert np.array_equal(c.cpu().numpy(), rc)
    assert np.array_equal(o.cpu().numpy(), ro)
    n = int(ro[-1])
    assert np.array_equal(sp.cpu().numpy()[:n], rsp)
    assert np.array_equal(pp.cpu().numpy(), rpp)


# ------------------------------------------------------------------------------------------- gather / combine
@pytest.mark.parametrize("dt", ["f16", "bf16"])
def test_gather_combine(dt):
    rng = np.random.default_rng(5)
    T, k, E, H = 33, 4, 16, 7168
    ids = np.stack([rng.permutation(E)[:k] for _ in range(T)]).astype(np.int32)
    x = O.round_act(rng.standard_normal((T, H)).astype(np.float32) * 0.5, dt)
    ops = _ops()
    c, o, sp, pp = ops.moe_permute(torch.from_numpy(ids).cuda(), E)
    xp = ops.moe_gather(_to_dev_act(x, dt), sp, k)
    _, _, rsp, rpp = O.moe_permute(ids, E)
    assert np.array_equal(_from_dev_act(xp, dt), x[rsp // k])
    yp = O.round_act(rng.standard_normal((T * k, H)).astype(np.float32), dt)
    w = rng.uniform(0, 1, (T, k)).astype(np.float32)
    y = ops.moe_combine(_to_dev_act(yp, dt), pp, torch.from_numpy(w).cuda())
    want = np.zeros((T, H), np.float32)
    for j in range(k):
        want += w[:, j:j + 1] * yp[rpp.reshape(T, k)[:, j]]
    np.testing.assert_allclose(_from_dev_act(y, dt), O.round_act(want, dt), rtol=RTOL, atol=ATOL)


@pytest.mark.parametrize("dt", ["f16", "bf16"])
def test_group_sums(dt):
    """(C, S) per (k-group, row): S = sum x, C = sum c_k x with the decode dequant's offsets."""
    rng = np.random.default_rng(9)
    T, k, E, H = 21, 3, 8, 1024
    ids = np.stack([rng.permutation(E)[:k] for _ in range(T)]).astype(np.int32)
    x = O.round_act(rng.standard_normal((T, H)).astype(np.float32) * 0.5, dt)
    ops = _ops()
    c, o, sp, pp = ops.moe_permute(torch.from_numpy(ids).cuda(), E)
    xp, xs = ops.moe_gather_sums(_to_dev_act(x, dt), sp, k)
    _, _, rsp, _ = O.moe_permute(ids, E)
    xr = x[rsp // k]
    assert np.array_equal(_from_dev_act(xp, dt), xr)
    want = O.group_sums(xr, dt)                     # [H/128][rows][2]
    got = xs.cpu().numpy()[:, :xr.shape[0], :]
    np.testing.assert_allclose(got, want, rtol=1e-5, atol=1e-3)
    got2 = ops.group_sums(xp).cpu().numpy()[:, :xr.shape[0], :]
    np.testing.assert_array_equal(got2, got)


# ------------------------------------------------------------------------------------------- grouped GEMM
def _gemm_case(dt, gated, counts, K, N, ntok, seed=0, sums=False, splitk=False):
    rng = np.random.default_rng(seed)
    E = len(counts)
    rows = int(sum(counts))
    q, z, s = O.synth_awq_expert_weights(rng, E, 2 * N if gated else N, K, dt)
    w = _packed(q, z, s, dt, gated)
    x = O.round_act(rng.standard_normal((rows, K)).astype(np.float32) * 0.5, dt)
    cnt = np.asarray(counts, np.int32)
    off = np.zeros(E + 1, np.int32)
    np.cumsum(cnt, out=off[1:])
    xd = _to_dev_act(x, dt)
    xs = _ops().group_sums(xd) if sums else None
    ws = None
    if splitk:
        wsb = _ops().gemm_ws_bytes(rows, K, E, N, gated, ntok)
        assert wsb > 0, "expected a split-K plan"
        ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    out = _ops().grouped_gemm(xd, w.blocks, E, N, gated, torch.from_numpy(cnt).cuda(),
                              torch.from_numpy(off).cuda(), ntok, xsum=xs, workspace=ws)
    torch.cuda.synchronize()
    want = O.grouped_gemm(x, O.dequant(q, z, s, dt), cnt, off, dt, gated)
    return _from_dev_act(out, dt), want


@pytest.mark.parametrize("ntok", [16, 32, 64, 128])
@pytest.mark.parametrize("gated", [False, True])
@pytest.mark.parametrize("sums", [False, True])
@pytest.mark.parametrize("K", [512, 384])  # k-pair (even K/128) and plain (odd) block modes
def test_grouped_gemm_f16(ntok, gated, sums, K):
    got, want = _gemm_case("f16", gated, [5, 0, 17, 1, 40, 130], K=K, N=256, ntok=ntok, sums=sums)
    np.testing.assert_allclose(got, want, rtol=RTOL, atol=ATOL)


@pytest.mark.parametrize("gated", [False, True])
@pytest.mark.parametrize("sums", [False, True])
@pytest.mark.parametrize("K", [384, 512])
def test_grouped_gemm_bf16(gated, sums, K):
    got, want = _gemm_case("bf16", gated, [3, 16, 0, 33], K=K, N=384, ntok=16, sums=sums)
    np.testing.assert_allclose(got, want, rtol=RTOL, atol=2 * ATOL)


@pytest.mark.parametrize("gated", [False, True])
@pytest.mark.parametrize("sums", [False, True])
def test_grouped_gemm_ring_wrap(gated, sums):
    """Enough tiles that every CTA runs several long tiles: the smem / TMEM rings wrap many times."""
    rng = np.random.default_rng(11)
    counts = list(rng.integers(1, 5, size=40))
    got, want = _gemm_case("f16", gated, counts, K=2048, N=1024, ntok=16, seed=12, sums=sums)
    np.testing.assert_allclose(got, want, rtol=RTOL, atol=ATOL)


@pytest.mark.parametrize("N,ntok", [(384, 16), (640, 16), (384, 32)])
@pytest.mark.parametrize("dt", ["f16", "bf16"])
def test_grouped_gemm_odd_ntiles_decode(N, ntok, dt):
    """An odd number of n-tiles cannot form n-pairs: the decode down projection falls back to k-pair
    stages (two k-groups of one n-tile per stage)."""
    got, want = _gemm_case(dt, False, [3, 0, 17, 9], K=1024, N=N, ntok=ntok, seed=9, sums=True)
    np.testing.assert_allclose(got, want, rtol=RTOL, atol=ATOL)


@pytest.mark.parametrize("gated,K,N", [(True, 2048, 1024), (False, 4096, 512), (False, 1920, 256)])
@pytest.mark.parametrize("dt", ["f16", "bf16"])
def test_grouped_gemm_splitk(gated, K, N, dt):
    """Few tiles (1-2 experts, a few tokens): the decode GEMM splits K over CTAs into fp32 partials
    and a finalize kernel (gated and n-pair block modes; K/128 = 15 is odd)."""
    got, want = _gemm_case(dt, gated, [2, 0, 3] if gated else [1, 2], K=K, N=N, ntok=16, seed=8, sums=True,
                           splitk=True)
    np.testing.assert_allclose(got, want, rtol=RTOL, atol=(2 if dt == "bf16" else 1) * ATOL)


@pytest.mark.parametrize("gated,K,N", [(True, 1024, 256), (False, 2048, 512), (False, 1024, 384)])
@pytest.mark.parametrize("dt", ["f16", "bf16"])
def test_grouped_gemm_offset_32(gated, K, N, dt, monkeypatch):
    """W4A16_DECODE_MAX_NTOK=32 (read per call): 32-token tiles in offset-code mode -- gate/up,
    n-pair down and (odd n-tile count) k-pair down kernels -- against the oracle."""
    monkeypatch.setenv("W4A16_DECODE_MAX_NTOK", "32")
    assert _ops().decode_max_ntok() == 32
    got, want = _gemm_case(dt, gated, [20, 0, 32, 7, 45], K=K, N=N, ntok=32, seed=12, sums=True)
    np.testing.assert_allclose(got, want, rtol=RTOL, atol=(2 if dt == "bf16" else 1) * ATOL)


@pytest.mark.parametrize("splitk", [False, True])
def test_gate_up_output_sums(splitk):
    """The gated GEMM also emits its output's (C, S) group sums (fused in the decode epilogue, or a
    sums pass after split-K): equal to group_sums of the output."""
    rng = np.random.default_rng(31)
    E, N, K, dt = 3, 1024, 2048, "f16"
    counts = [2, 0, 3] if splitk else [5, 16, 9]
    q, z, s = O.synth_awq_expert_weights(rng, E, 2 * N, K, dt)
    w = _packed(q, z, s, dt, True)
    rows = int(sum(counts))
    cnt = np.asarray(counts, np.int32)
    off = np.zeros(E + 1, np.int32)
    np.cumsum(cnt, out=off[1:])
    xd = _to_dev_act(O.round_act(rng.standard_normal((rows, K)).astype(np.float32) * 0.5, dt), dt)
    ops = _ops()
    xs = ops.group_sums(xd)
    hs = torch.full(ops.sums_shape(rows, N), float("nan"), dtype=torch.float32, device="cuda")
    wsb = ops.gemm_ws_bytes(rows, K, E, N, True, 16)
    assert wsb > 0  # few tiles: a split is planned; without a workspace the fused epilogue path runs
    ws = torch.zeros(wsb, dtype=torch.uint8, device="cuda") if splitk else None
    h = ops.grouped_gemm(xd, w.blocks, E, N, True, torch.from_numpy(cnt).cuda(), torch.from_numpy(off).cuda(), 16,
                         xsum=xs, workspace=ws, osum=hs)
    want = ops.group_sums(h).cpu().numpy()[:, :rows]
    got = hs.cpu().numpy()[:, :rows]
    np.testing.assert_allclose(got, want, rtol=1e-5, atol=2e-2)


def test_grouped_gemm_decode_shapes():
    """DeepSeek-R1 down-projection shape (K=2048 -> 8 k-pair stages per tile) in decode mode."""
    got, want = _gemm_case("f16", False, [2, 1, 3, 0, 2], K=2048, N=512, ntok=16, seed=4, sums=True)
    np.testing.assert_allclose(got, want, rtol=RTOL, atol=ATOL)


def test_dense_w4a16_linear():
    """Config 1 shape: M=16, N=K=1024, one expert."""
    got, want = _gemm_case("f16", False, [16], K=1024, N=1024, ntok=16, seed=3, sums=True)
    np.testing.assert_allclose(got, want, rtol=RTOL, atol=ATOL)


@pytest.mark.parametrize("M", [1, 16, 200])
def test_dense_w4a16_linear_llama_shape(M):
    """BASELINE config 2: Llama-3-8B linear K=4096, N=14336 through the public dense entry point
    (decode mode + split-K at small M, scale-in-dequant at larger M)."""
    from paper_2504_16214_b200.moe import w4a16_linear
    rng = np.random.default_rng(M)
    N, K = 14336, 4096
    q, z, s = O.synth_awq_expert_weights(rng, 1, N, K, "f16")
    w = _packed(q, z, s, "f16", False)
    x = O.round_act(rng.standard_normal((M, K)).astype(np.float32) * 0.5, "f16")
    got = _from_dev_act(w4a16_linear(_to_dev_act(x, "f16"), w), "f16")
    torch.cuda.synchronize()
    want = O.round_act(x @ O.dequant(q, z, s, "f16")[0].T, "f16")
    np.testing.assert_allclose(got, want, rtol=RTOL, atol=ATOL)


# ------------------------------------------------------------------------------------------- layer
@pytest.mark.parametrize("T,E,k", [(0, 8, 2), (7, 1, 1), (33, 4, 4), (5, 1024, 8)])
def test_moe_layer_edge_shapes(T, E, k):
    """Edge shapes: an empty batch, a single expert with top-1, every token on every expert (k = E),
    and the largest expert count (1024, most experts empty)."""
    from paper_2504_16214_b200.moe import fused_moe_w4a16
    from paper_2504_16214_b200.moe.weights import MoEWeights
    rng = np.random.default_rng(E + k)
    H, I, dt = 128, 128, "f16"
    q13, z13, s13 = O.synth_awq_expert_weights(rng, E, 2 * I, H, dt)
    q2, z2, s2 = O.synth_awq_expert_weights(rng, E, H, I, dt)
    w = MoEWeights(_packed(q13, z13, s13, dt, True), _packed(q2, z2, s2, dt, False))
    x = O.round_act(rng.standard_normal((T, H)).astype(np.float32) * 0.5, dt)
    lg = rng.standard_normal((T, E)).astype(np.float32)
    y = fused_moe_w4a16(_to_dev_act(x, dt), torch.from_numpy(lg).cuda(), w, k, "softmax", True)
    torch.cuda.synchronize()
    assert tuple(y.shape) == (T, H)
    if T:
        ids, wts = O.route_topk(lg, k, "softmax", True)
        want = O.moe_forward(x, O.dequant(q13, z13, s13, dt), O.dequant(q2, z2, s2, dt), ids, wts, dt)
        np.testing.assert_allclose(_from_dev_act(y, dt), want, rtol=RTOL, atol=ATOL)


@pytest.mark.parametrize("dt", ["f16", "bf16"])
@pytest.mark.parametrize("T,E,k,H,I", [(1, 8, 2, 256, 384), (24, 16, 4, 512, 256), (130, 8, 2, 256, 256),
                                       (64, 32, 8, 256, 128)])
def test_moe_layer(dt, T, E, k, H, I):
    from paper_2504_16214_b200.moe import moe_w4a16, select_experts
    from paper_2504_16214_b200.moe.weights import MoEWeights
    rng = np.random.default_rng(T + E)
    q13, z13, s13 = O.synth_awq_expert_weights(rng, E, 2 * I, H, dt)
    q2, z2, s2 = O.synth_awq_expert_weights(rng, E, H, I, dt)
    weights = MoEWeights(_packed(q13, z13, s13, dt, True), _packed(q2, z2, s2, dt, False))
    x = O.round_act(rng.standard_normal((T, H)).astype(np.float32) * 0.5, dt)
    lg = rng.standard_normal((T, E)).astype(np.float32)
    wts, ids = select_experts(torch.from_numpy(lg).cuda(), k, "softmax", True)
    y = moe_w4a16(_to_dev_act(x, dt), weights, wts, ids)
    torch.cuda.synchronize()
    rid, rw = O.route_topk(lg, k, "softmax", True)
    assert np.array_equal(ids.cpu().numpy(), rid)
    want = O.moe_forward(x, O.dequant(q13, z13, s13, dt), O.dequant(q2, z2, s2, dt), rid, rw, dt)
    np.testing.assert_allclose(_from_dev_act(y, dt), want, rtol=RTOL, atol=ATOL)


def test_fused_moe_graph_matches_eager():
    """The CUDA-graph-captured layer replays the same kernels: identical output to the eager call,
    and new inputs copied into the graph take effect."""
    from paper_2504_16214_b200.moe import FusedMoEGraph, fused_moe_w4a16
    from paper_2504_16214_b200.moe.weights import MoEWeights
    rng = np.random.default_rng(21)
    T, E, k, H, I, dt = 12, 16, 4, 512, 256, "f16"
    q13, z13, s13 = O.synth_awq_expert_weights(rng, E, 2 * I, H, dt)
    q2, z2, s2 = O.synth_awq_expert_weights(rng, E, H, I, dt)
    weights = MoEWeights(_packed(q13, z13, s13, dt, True), _packed(q2, z2, s2, dt, False))
    g = FusedMoEGraph(weights, T, k, "softmax", True, torch.float16)
    for seed in (1, 2):
        r = np.random.default_rng(seed)
        x = _to_dev_act(O.round_act(r.standard_normal((T, H)).astype(np.float32) * 0.5, dt), dt)
        lg = torch.from_numpy(r.standard_normal((T, E)).astype(np.float32)).cuda()
        want = fused_moe_w4a16(x, lg, weights, k, "softmax", True).clone()
        got = g(x, lg)
        torch.cuda.synchronize()
        assert torch.equal(got, want)


def test_fused_moe_pipeline_matches_eager():
    """The copy-overlapped serving loop (two graph slots, H2D / D2H streams): every step's host output
    equals the eager layer on that step's host inputs, across slot reuse."""
    from paper_2504_16214_b200.moe import FusedMoEPipeline, fused_moe_w4a16
    from paper_2504_16214_b200.moe.weights import MoEWeights
    rng = np.random.default_rng(22)
    T, E, k, H, I, dt = 12, 16, 4, 512, 256, "f16"
    q13, z13, s13 = O.synth_awq_expert_weights(rng, E, 2 * I, H, dt)
    q2, z2, s2 = O.synth_awq_expert_weights(rng, E, H, I, dt)
    weights = MoEWeights(_packed(q13, z13, s13, dt, True), _packed(q2, z2, s2, dt, False))
    pipe = FusedMoEPipeline(weights, T, k, "softmax", True, torch.float16)
    xs, lgs, ys = [], [], []
    for seed in range(5):
        r = np.random.default_rng(100 + seed)
        xs.append(_to_dev_act(O.round_act(r.standard_normal((T, H)).astype(np.float32) * 0.5, dt), dt).cpu().pin_memory())
        lgs.append(torch.from_numpy(r.standard_normal((T, E)).astype(np.float32)).pin_memory())
        ys.append(torch.empty((T, H), dtype=torch.float16).pin_memory())
    pipe.start()
    for x, lg, y in zip(xs, lgs, ys):
        pipe(x, lg, y)
    pipe.finish()
    torch.cuda.synchronize()
    for x, lg, y in zip(xs, lgs, ys):
        want = fused_moe_w4a16(x.cuda(), lg.cuda(), weights, k, "softmax", True).cpu()
        assert torch.equal(y, want)


@pytest.mark.parametrize("world,el", [(1, 256), (2, 128), (8, 32), (4, 3)])
def test_ep_local_order(world, el):
    """Receiver-side local-expert order from the received counts == ids + stable permutation."""
    from paper_2504_16214_b200.moe.ep import local_expert_ids
    rng = np.random.default_rng(world * 100 + el)
    cnt = rng.integers(0, 6, size=(world, el)).astype(np.int32)
    cnt[0, 0] = 0
    n = int(cnt.sum())
    rc = torch.from_numpy(cnt).cuda()
    got = _ops().ep_local_order(rc, n)
    lid = local_expert_ids(rc, n).cpu().numpy()
    want = O.moe_permute(lid, el)
    for g, w in zip(got, want):
        assert np.array_equal(g.cpu().numpy()[:len(w)], w)


@pytest.mark.parametrize("ntok,splitk", [(16, False), (16, True), (64, False)])
def test_grouped_gemm_out_rows(ntok, splitk):
    """out_rows scatters result rows (the EP down GEMM writes arrival order directly): equals the
    plain output permuted."""
    rng = np.random.default_rng(41)
    E, N, K, dt = 2, 512, 1024, "f16"
    counts = [3, 2] if ntok == 16 else [40, 30]
    q, z, s = O.synth_awq_expert_weights(rng, E, N, K, dt)
    w = _packed(q, z, s, dt, False)
    rows = int(sum(counts))
    cnt = torch.tensor(counts, dtype=torch.int32).cuda()
    off = torch.tensor([0, counts[0], rows], dtype=torch.int32).cuda()
    xd = _to_dev_act(O.round_act(rng.standard_normal((rows, K)).astype(np.float32) * 0.5, dt), dt)
    ops = _ops()
    xs = ops.group_sums(xd) if ntok == 16 else None
    wsb = ops.gemm_ws_bytes(rows, K, E, N, False, ntok) if splitk else 0
    ws = torch.zeros(wsb, dtype=torch.uint8, device="cuda") if wsb else None
    perm = torch.from_numpy(rng.permutation(rows).astype(np.int32)).cuda()
    plain = ops.grouped_gemm(xd, w.blocks, E, N, False, cnt, off, ntok, xsum=xs, workspace=ws)
    scat = ops.grouped_gemm(xd, w.blocks, E, N, False, cnt, off, ntok, xsum=xs, workspace=ws, out_rows=perm)
    torch.cuda.synchronize()
    assert torch.equal(scat[perm.long()], plain)


@pytest.mark.parametrize("T", [3, 40, 600])
def test_c_abi_moe_forward(T):
    """The one-call C entry point w4a16_moe_forward (caller workspace, precomputed routing) through
    ctypes == the oracle layer (decode, 32/64-token and split-K plans depending on T)."""
    import ctypes
    from paper_2504_16214_b200.moe import _lib
    from paper_2504_16214_b200.moe.weights import MoEWeights
    lib = _lib.load()
    lib.w4a16_moe_workspace_bytes.restype = ctypes.c_int64
    lib.w4a16_moe_workspace_bytes.argtypes = [ctypes.c_int64] * 5
    lib.w4a16_moe_forward.restype = ctypes.c_int
    p, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
    lib.w4a16_moe_forward.argtypes = [p, i64, i64, i64, i64, i64, p, p, p, p, i32, p, p, i64, p]
    rng = np.random.default_rng(T)
    E, k, H, I, dt = 16, 4, 512, 256, "f16"
    q13, z13, s13 = O.synth_awq_expert_weights(rng, E, 2 * I, H, dt)
    q2, z2, s2 = O.synth_awq_expert_weights(rng, E, H, I, dt)
    w = MoEWeights(_packed(q13, z13, s13, dt, True), _packed(q2, z2, s2, dt, False))
    x = O.round_act(rng.standard_normal((T, H)).astype(np.float32) * 0.5, dt)
    lg = rng.standard_normal((T, E)).astype(np.float32)
    ids, wts = O.route_topk(lg, k, "softmax", True)
    xd = _to_dev_act(x, dt)
    idd, wd = torch.from_numpy(ids).cuda(), torch.from_numpy(wts).cuda()
    y = torch.empty_like(xd)
    wsb = lib.w4a16_moe_workspace_bytes(T, k, E, H, I)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    rc = lib.w4a16_moe_forward(xd.data_ptr(), T, H, I, E, k, idd.data_ptr(), wd.data_ptr(), w.w13.blocks.data_ptr(),
                               w.w2.blocks.data_ptr(), 0, y.data_ptr(), ws.data_ptr(), wsb,
                               torch.cuda.current_stream().cuda_stream)
    assert rc == 0
    torch.cuda.synchronize()
    want = O.moe_forward(x, O.dequant(q13, z13, s13, dt), O.dequant(q2, z2, s2, dt), ids, wts, dt)
    np.testing.assert_allclose(_from_dev_act(y, dt), want, rtol=RTOL, atol=ATOL)
    assert lib.w4a16_moe_forward(xd.data_ptr(), T, H, I, E, k, idd.data_ptr(), wd.data_ptr(), w.w13.blocks.data_ptr(),
                                 w.w2.blocks.data_ptr(), 0, y.data_ptr(), ws.data_ptr(), wsb - 1,
                                 torch.cuda.current_stream().cuda_stream) == -6  # W4_ERR_WORKSPACE


@pytest.mark.parametrize("T,dt", [(20, "f16"), (300, "bf16")])
def test_fused_moe_shared_expert(T, dt):
    """DeepSeek-style shared expert (always active, weight 1) packed as the last expert: the layer ==
    routed oracle layer + the shared expert's MLP on every token; also through the CUDA graph."""
    from paper_2504_16214_b200.moe import FusedMoEGraph, fused_moe_w4a16
    from paper_2504_16214_b200.moe.weights import MoEWeights
    rng = np.random.default_rng(T)
    E, k, H, I = 16, 4, 256, 256  # 16 routed + 1 shared
    q13, z13, s13 = O.synth_awq_expert_weights(rng, E + 1, 2 * I, H, dt)
    q2, z2, s2 = O.synth_awq_expert_weights(rng, E + 1, H, I, dt)
    w = MoEWeights(_packed(q13, z13, s13, dt, True), _packed(q2, z2, s2, dt, False))
    x = O.round_act(rng.standard_normal((T, H)).astype(np.float32) * 0.5, dt)
    lg = rng.standard_normal((T, E)).astype(np.float32)
    y = fused_moe_w4a16(_to_dev_act(x, dt), torch.from_numpy(lg).cuda(), w, k, "sigmoid", True, num_expert_group=4,
                        topk_group=2, routed_scaling_factor=2.5, num_shared_experts=1)
    torch.cuda.synchronize()
    rid, rw = O.grouped_topk(lg, k, 4, 2, "sigmoid", True, None, 2.5)
    ids = np.concatenate([rid, np.full((T, 1), E, np.int32)], axis=1)
    wts = np.concatenate([rw, np.ones((T, 1), np.float32)], axis=1)
    want = O.moe_forward(x, O.dequant(q13, z13, s13, dt), O.dequant(q2, z2, s2, dt), ids, wts, dt)
    tol = (2 if dt == "bf16" else 1) * ATOL
    np.testing.assert_allclose(_from_dev_act(y, dt), want, rtol=RTOL, atol=tol)
    if dt == "f16":  # graph replay of the same layer (softmax routing here)
        g = FusedMoEGraph(w, T, k, "softmax", True, torch.float16, num_shared_experts=1)
        y2 = g(_to_dev_act(x, dt), torch.from_numpy(lg).cuda())
        torch.cuda.synchronize()
        rid, rw = O.route_topk(lg, k, "softmax", True)
        ids = np.concatenate([rid, np.full((T, 1), E, np.int32)], axis=1)
        wts = np.concatenate([rw, np.ones((T, 1), np.float32)], axis=1)
        want2 = O.moe_forward(x, O.dequant(q13, z13, s13, dt), O.dequant(q2, z2, s2, dt), ids, wts, dt)
        np.testing.assert_allclose(_from_dev_act(y2, dt), want2, rtol=RTOL, atol=tol)


@pytest.mark.parametrize("ntok,dt", [(16, "f16"), (16, "bf16"), (32, "f16"), (64, "bf16"), (128, "f16")])
def test_grouped_gemm_fused_gather(ntok, dt):
    """The gate/up GEMM gathering x's rows itself (TMA gather4 in the producer) == gather kernel +
    GEMM, bit for bit (same rows, same sums, same kernel otherwise)."""
    ops = _ops()
    rng = np.random.default_rng(ntok)
    T, E, k, K, N = 150, 12, 4, 512, 256
    q, z, s = O.synth_awq_expert_weights(rng, E, 2 * N, K, dt)
    w = _packed(q, z, s, dt, True)
    x = _to_dev_act(O.round_act(rng.standard_normal((T, K)).astype(np.float32) * 0.5, dt), dt)
    ids = torch.from_numpy(np.stack([rng.permutation(E)[:k] for _ in range(T)]).astype(np.int32)).cuda()
    c, o, sp, pp = ops.moe_permute(ids, E)
    P = T * k
    decode = ntok == 16
    if decode:
        xp, xsp = ops.moe_gather_sums(x, sp, k)
        xs = ops.group_sums(x)
    else:
        xp, xsp, xs = ops.moe_gather(x, sp, k, P), None, None
    want = ops.grouped_gemm(xp, w.blocks, E, N, True, c, o, ntok, xsum=xsp)
    got = ops.grouped_gemm_gather(x, sp, k, w.blocks, E, N, True, c, o, ntok, xsum=xs, rows=P)
    torch.cuda.synchronize()
    assert torch.equal(got, want)


def test_ep_nccl_world1_layer():
    """The expert-parallel path over NCCL (all-gather dispatch, local experts with the fp32 partial
    combine, reduce-scatter + rounding) at world size 1 == the oracle layer; eager, CUDA-graph
    captured (the NCCL collectives inside the graph), and through the one-call C entry
    w4a16_moe_forward_ep with a communicator made by w4a16_ep_unique_id / w4a16_ep_comm_init."""
    import socket
    import torch.distributed as dist
    from paper_2504_16214_b200.moe import fused_moe_w4a16
    from paper_2504_16214_b200.moe.weights import MoEWeights
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        rng = np.random.default_rng(41)
        for T, dt in ((40, "f16"), (300, "bf16")):  # decode (16-token tiles) and prefill tiles
            E, k, H, I = 16, 4, 256, 256
            q13, z13, s13 = O.synth_awq_expert_weights(rng, E, 2 * I, H, dt)
            q2, z2, s2 = O.synth_awq_expert_weights(rng, E, H, I, dt)
            w = MoEWeights(_packed(q13, z13, s13, dt, True), _packed(q2, z2, s2, dt, False))
            x = O.round_act(rng.standard_normal((T, H)).astype(np.float32) * 0.5, dt)
            lg = rng.standard_normal((T, E)).astype(np.float32)
            y = fused_moe_w4a16(_to_dev_act(x, dt), torch.from_numpy(lg).cuda(), w, k, "softmax", True,
                                ep_group=dist.group.WORLD)
            torch.cuda.synchronize()
            rid, rw = O.route_topk(lg, k, "softmax", True)
            want = O.moe_forward(x, O.dequant(q13, z13, s13, dt), O.dequant(q2, z2, s2, dt), rid, rw, dt)
            np.testing.assert_allclose(_from_dev_act(y, dt), want, rtol=RTOL, atol=(2 if dt == "bf16" else 1) * ATOL)
            if dt == "f16":  # the same EP layer captured in a CUDA graph (no host sync anywhere in the step)
                from paper_2504_16214_b200.moe import FusedMoEGraph
                g = FusedMoEGraph(w, T, k, "softmax", True, torch.float16, ep_group=dist.group.WORLD)
                yg = g(_to_dev_act(x, dt), torch.from_numpy(lg).cuda())
                torch.cuda.synchronize()
                assert torch.equal(yg, y)
                _ep_c_abi_world1(w, x, rid, rw, want, dt)
        # a shared expert (packed last): routed experts through the exchange, the shared one locally
        T, E, k, H, I, dt = 24, 8, 2, 256, 256, "f16"
        q13, z13, s13 = O.synth_awq_expert_weights(rng, E + 1, 2 * I, H, dt)
        q2, z2, s2 = O.synth_awq_expert_weights(rng, E + 1, H, I, dt)
        w = MoEWeights(_packed(q13, z13, s13, dt, True), _packed(q2, z2, s2, dt, False))
        x = O.round_act(rng.standard_normal((T, H)).astype(np.float32) * 0.5, dt)
        lg = rng.standard_normal((T, E)).astype(np.float32)
        from paper_2504_16214_b200.moe.ep import shard_with_shared
        routed, shared = shard_with_shared(w, 1, dist.get_world_size(), dist.get_rank())
        y = fused_moe_w4a16(_to_dev_act(x, dt), torch.from_numpy(lg).cuda(), routed, k, "softmax", True,
                            ep_group=dist.group.WORLD, shared_weights=shared)
        torch.cuda.synchronize()
        rid, rw = O.route_topk(lg, k, "softmax", True)
        ids = np.concatenate([rid, np.full((T, 1), E, np.int32)], axis=1)
        wts = np.concatenate([rw, np.ones((T, 1), np.float32)], axis=1)
        want = O.moe_forward(x, O.dequant(q13, z13, s13, dt), O.dequant(q2, z2, s2, dt), ids, wts, dt)
        # the EP sum adds two rounded partial outputs (routed + shared): one extra rounding
        np.testing.assert_allclose(_from_dev_act(y, dt), want, rtol=RTOL, atol=2 * ATOL)
    finally:
        dist.destroy_process_group()


def _ep_c_abi_world1(w, x, ids, wts, want, dt):
    """w4a16_moe_forward_ep through ctypes on a library-made NCCL communicator of one rank."""
    import ctypes
    from paper_2504_16214_b200.moe import _lib
    lib = _lib.load()
    assert lib.w4a16_ep_available() == 1
    uid = (ctypes.c_uint8 * 128)()
    assert lib.w4a16_ep_unique_id(ctypes.addressof(uid)) == 0
    comm = ctypes.c_void_p()
    assert lib.w4a16_ep_comm_init(ctypes.addressof(uid), 0, 1, ctypes.byref(comm)) == 0
    try:
        assert (lib.w4a16_ep_comm_rank(comm), lib.w4a16_ep_comm_size(comm)) == (0, 1)
        T, H = x.shape
        E, k, I = w.num_experts, ids.shape[1], w.inter
        wsb = lib.w4a16_moe_ep_workspace_bytes(T, 1, k, E, H, I)
        ws = torch.zeros(wsb, dtype=torch.uint8, device="cuda")
        xd = _to_dev_act(x, dt)
        y = torch.empty_like(xd)
        idd, wd = torch.from_numpy(ids).cuda(), torch.from_numpy(wts).cuda()
        rc = lib.w4a16_moe_forward_ep(comm, xd.data_ptr(), T, H, I, E, k, idd.data_ptr(), wd.data_ptr(),
                                      w.w13.blocks.data_ptr(), w.w2.blocks.data_ptr(), 0 if dt == "f16" else 1,
                                      y.data_ptr(), ws.data_ptr(), wsb, torch.cuda.current_stream().cuda_stream)
        assert rc == 0
        torch.cuda.synchronize()
        np.testing.assert_allclose(_from_dev_act(y, dt), want, rtol=RTOL, atol=ATOL)
    finally:
        assert lib.w4a16_ep_comm_destroy(comm) == 0


@pytest.mark.parametrize("dt", ["f16", "bf16"])
def test_combine_f32_and_localize(dt):
    """The expert-parallel building blocks: the fp32 (unrounded) combine rounds to the regular
    combine bit for bit, and ep_localize keeps exactly the ids of one shard (others -> -1)."""
    ops = _ops()
    rng = np.random.default_rng(5)
    T, k, H, E = 37, 8, 512, 64
    ids = torch.from_numpy(np.stack([rng.permutation(E)[:k] for _ in range(T)]).astype(np.int32)).cuda()
    ids[3, 2] = -1
    w = torch.from_numpy(rng.random((T, k)).astype(np.float32)).cuda()
    c, o, sp, pp = ops.moe_permute(ids, E)
    tdt = torch.float16 if dt == "f16" else torch.bfloat16
    yp = (torch.randn((T * k, H), device="cuda") * 0.5).to(tdt)
    y = ops.moe_combine(yp, pp, w)
    y32 = ops.moe_combine(yp, pp, w, f32=True)
    torch.cuda.synchronize()
    assert y32.dtype == torch.float32 and torch.equal(y32.to(tdt), y)
    for base, n in ((0, 64), (16, 16), (48, 32), (60, 8)):
        loc = ops.ep_localize(ids, base, n)
        want = torch.where((ids >= base) & (ids < base + n), ids - base, torch.full_like(ids, -1))
        assert torch.equal(loc, want)


def test_moe_w4a16_raw_awq_overload():
    """moe_w4a16(x, w13_q, w13_s, w13_z, w2_q, w2_s, w2_z, topk_weights, topk_ids, group_size=128)
    -- vLLM's AWQ MoE tensors, repacked on first use == the packed-weights call."""
    from paper_2504_16214_b200.moe import moe_w4a16
    from paper_2504_16214_b200.moe.weights import pack_moe_awq
    rng = np.random.default_rng(77)
    T, E, k, H, I, dt = 33, 8, 2, 256, 256, "bf16"
    q13, z13, s13 = O.synth_awq_expert_weights(rng, E, 2 * I, H, dt)
    q2, z2, s2 = O.synth_awq_expert_weights(rng, E, H, I, dt)
    tdt = torch.bfloat16
    awq = []
    for q, z, s in ((q13, z13, s13), (q2, z2, s2)):
        qw, sc, qz = O.to_awq(q, z, s)
        awq += [torch.from_numpy(qw).cuda(), torch.from_numpy(sc).cuda().to(tdt), torch.from_numpy(qz).cuda()]
    x = _to_dev_act(O.round_act(rng.standard_normal((T, H)).astype(np.float32) * 0.5, dt), dt)
    ids, wts = O.route_topk(rng.standard_normal((T, E)).astype(np.float32), k, "softmax", True)
    idd, wd = torch.from_numpy(ids).cuda(), torch.from_numpy(wts).cuda()
    y_raw = moe_w4a16(x, awq[0], awq[1], awq[2], awq[3], awq[4], awq[5], wd, idd, group_size=128)
    y_raw2 = moe_w4a16(x, *awq, wd, idd)  # cached repack
    y_pk = moe_w4a16(x, pack_moe_awq(*awq), wd, idd)
    torch.cuda.synchronize()
    assert torch.equal(y_raw, y_pk) and torch.equal(y_raw2, y_pk)


def test_empty_inputs_c_abi():
    """Empty batches through the routing / permutation entry points: OK without touching the (null)
    pair pointers; the permutation still zeroes the expert counts and offsets."""
    ops = _ops()
    E = 16
    lg = torch.empty((0, E), dtype=torch.float32, device="cuda")
    ids, w = ops.route_topk(lg, 4)
    assert ids.shape == (0, 4)
    c, o, sp, pp = ops.moe_permute(torch.empty((0, 4), dtype=torch.int32, device="cuda"), E)
    torch.cuda.synchronize()
    assert int(c.sum()) == 0 and int(o.abs().sum()) == 0
    ids, w, c, o, sp, pp = ops.route_permute(lg, 4)
    torch.cuda.synchronize()
    assert int(c.sum()) == 0 and int(o.abs().sum()) == 0


def test_against_vllm_kernels_golden():
    """The B200 path vs vLLM 0.22's own kernels on the same inputs (tests/golden/vllm_moe.npz from
    tools/make_golden_vllm.py): routing ids bit-exact with its CUDA topk_softmax / topk_sigmoid, the
    W4A16 layer within rtol / atol 1e-2 of its moe_wna16 Triton fused_experts."""
    from pathlib import Path
    from paper_2504_16214_b200.moe import moe_w4a16
    from paper_2504_16214_b200.moe.weights import MoEWeights
    d = np.load(Path(__file__).resolve().parent / "golden" / "vllm_moe.npz")
    ops = _ops()
    for ci in range(6):
        T, E, k, soft, rn = (int(v) for v in d[f"route{ci}_meta"])
        ids, w = ops.route_topk(torch.from_numpy(d[f"route{ci}_logits"]).cuda(), k, "softmax" if soft else "sigmoid",
                                bool(rn))
        assert np.array_equal(ids.cpu().numpy(), d[f"route{ci}_ids"])
        np.testing.assert_allclose(w.cpu().numpy(), d[f"route{ci}_w"], rtol=2e-6, atol=2e-7)
    for li in range(2):
        T, E, k, H, I, f16 = (int(v) for v in d[f"layer{li}_meta"])
        dt = "f16" if f16 else "bf16"
        g = lambda n: d[f"layer{li}_{n}"]  # noqa: E731
        wts = MoEWeights(_packed(g("q13"), g("z13"), g("s13"), dt, True), _packed(g("q2"), g("z2"), g("s2"), dt, False))
        y = moe_w4a16(_to_dev_act(g("x"), dt), wts, torch.from_numpy(g("w")).cuda(), torch.from_numpy(g("ids")).cuda())
        torch.cuda.synchronize()
        np.testing.assert_allclose(_from_dev_act(y, dt), g("y"), rtol=RTOL, atol=ATOL)
