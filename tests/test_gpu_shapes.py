"""GPU parity at the BASELINE.json shapes (north star: rtol 1e-2 / atol 1e-2, fp32 accumulate; routing
ids bit-exact), through the public API on full-size synthetic weights:

* DeepSeek-R1 MoE layer (E=256, k=8, H=7168, I=2048): decode T=1 and T=64, prefill T=8192, f16 and bf16,
  plus heavy-tailed activations (1 % of entries x50) at K=7168 in the decode (offset-code) mode;
* Mixtral-8x7B (E=8, k=2, H=4096, I=14336) at T=16 and T=2048;
* Qwen3-30B-A3B-style (E=128, k=8, H=2048, I=768) at T=256, uniform and Zipf(1.1)-skewed routing;
* the dense Llama-3-8B linear (K=4096, N=14336) at M=4096;
* a grouped GEMM whose row count passes 2^20 (tile-table packing limit).

Tolerance: |got - want| <= atol + rtol * scale with rtol = atol = 1e-2, where scale is the magnitude of
the terms each output sums, sum_j |w_j| * (|h_j| @ |W2_j|^T) (``moe_oracle.expert_rows``). At these K
(2048..14336) the pinned intermediate roundings (h and each expert's output in fp16/bf16) see 1-ulp
flips between any two fp32 accumulation orders; such a flip moves an output by ~ulp of those terms,
which for outputs that cancel to near zero exceeds 1e-2 of |want| (bf16 ulp at 32 is 0.25). The
fraction of elements that also meet the plain |want|-relative rule is asserted >= 99 % (fp16) / 90 %
(bf16, 8-bit mantissa).

The GPU always runs the WHOLE layer (every routed expert, the real tile plan). The CPU oracle then checks
a sample of experts: the routing weights of pairs routed to unsampled experts are zeroed, so the layer
output equals the oracle's restricted to the sampled experts (`moe_oracle.moe_forward_expertwise`). Each
sampled expert's AWQ tensors are regenerated from its own seed (`weights.random_awq_expert`)."""
import numpy as np
import pytest
import torch

import moe_oracle as O

pytestmark = pytest.mark.gpu

RTOL = 1e-2
ATOL = 1e-2
TDT = {"f16": torch.float16, "bf16": torch.bfloat16}


def _to_dev_act(a: np.ndarray, dt: str) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(O.act_bits(a, dt))).view(TDT[dt]).cuda()


def _from_dev_act(t: torch.Tensor, dt: str) -> np.ndarray:
    return O.bits_to_f32(t.view(torch.int16).cpu().numpy().view(np.uint16), dt)


def _expert_awq(seed: int, e: int, N: int, K: int, dt: str):
    from paper_2504_16214_b200.moe.weights import random_awq_expert
    qw, sc, qz = random_awq_expert(seed, e, N, K, TDT[dt], "cuda")
    sc_bits = sc.view(torch.int16).cpu().numpy().view(np.uint16)
    return O.from_awq(qw.cpu().numpy(), O.bits_to_f32(sc_bits, dt), qz.cpu().numpy())


def _sample_experts(ids: np.ndarray, E: int, n: int, rng) -> list[int]:
    """The most loaded experts (their m-tiles are the full / multi-tile ones), the least loaded
    touched ones (partial tiles) and random others, up to n."""
    counts = np.bincount(ids.ravel(), minlength=E)
    touched = np.nonzero(counts)[0]
    if len(touched) <= n:
        return sorted(int(e) for e in touched)
    order = touched[np.argsort(-counts[touched], kind="stable")]
    pick = list(order[: n // 3]) + list(order[::-1][: n // 3])
    rest = [e for e in touched if e not in pick]
    pick += list(rng.choice(rest, size=n - len(pick), replace=False))
    return sorted(int(e) for e in pick)


def _layer_case(E, k, H, I, T, dt, n_check, seed, zipf=False, outliers=False, graph=False):
    from paper_2504_16214_b200.moe import FusedMoEGraph, moe_w4a16, random_moe_weights, select_experts
    rng = np.random.default_rng(seed)
    weights = random_moe_weights(E, H, I, TDT[dt], device="cuda", seed=seed)
    x = rng.standard_normal((T, H)).astype(np.float32) * 0.5
    if outliers:  # heavy tail: 1 % of the entries x50 (activation outlier channels / tokens)
        x[rng.random((T, H)) < 0.01] *= 50.0
    x = O.round_act(x, dt)
    lg = rng.standard_normal((T, E)).astype(np.float32)
    if zipf:  # expert popularity ~ Zipf(1.1) over a random expert order (logit bias = log p)
        lg += (-1.1 * np.log(rng.permutation(E) + 1.0)).astype(np.float32)
    lgd = torch.from_numpy(lg).cuda()
    wts, ids = select_experts(lgd, k, "softmax", True)
    rid, rw = O.route_topk(lg, k, "softmax", True)
    assert np.array_equal(ids.cpu().numpy(), rid)  # routing: bit-exact
    np.testing.assert_allclose(wts.cpu().numpy(), rw, rtol=1e-5, atol=1e-6)
    pick = _sample_experts(rid, E, n_check, rng)
    keep = np.isin(rid, pick)
    w_masked = np.where(keep, rw, 0.0).astype(np.float32)
    xd = _to_dev_act(x, dt)
    if graph:  # the CUDA-graph path the bench times (routing inside; weights can't be masked there)
        g = FusedMoEGraph(weights, T, k, "softmax", True, TDT[dt], x=xd, router_logits=lgd)
        torch.testing.assert_close(g(xd, lgd), moe_w4a16(xd, weights, wts, ids), rtol=0, atol=0)
    y = moe_w4a16(xd, weights, torch.from_numpy(w_masked).cuda(), ids)
    got = _from_dev_act(y, dt)
    torch.cuda.synchronize()
    # oracle over the sampled experts only (ids remapped to the sample, others dropped)
    local = {e: i for i, e in enumerate(pick)}
    ids_loc = np.vectorize(lambda e: local.get(int(e), -1))(rid).astype(np.int32)
    w13 = [_expert_awq(2 * seed, e, 2 * I, H, dt) for e in pick]
    w2 = [_expert_awq(2 * seed + 1, e, H, I, dt) for e in pick]
    st = lambda ws, i: np.stack([w[i] for w in ws])  # noqa: E731
    from paper_2504_16214_b200.moe import ops
    decode = ops.pick_ntok(T * k, E) <= ops.decode_max_ntok()  # offset-code GEMMs: unrounded (q - z) * s
    want, scale = O.moe_forward_expertwise(x, st(w13, 0), st(w13, 1), st(w13, 2), st(w2, 0), st(w2, 1), st(w2, 2),
                                           ids_loc, w_masked, dt, with_scale=True, exact_dequant=decode)
    return got, want, scale, pick


def _check(got, want, scale, plain_frac=0.99):
    err = np.abs(got - want)
    bad = err > ATOL + RTOL * scale
    assert not bad.any(), (f"{int(bad.sum())} of {bad.size} outputs off: max |diff| {err.max():.4g}, "
                           f"worst at scale {scale.flat[int(np.argmax(err - RTOL * scale))]:.4g}")
    plain = np.mean(err <= ATOL + RTOL * np.abs(want))
    assert plain >= plain_frac, f"only {plain:.4%} within the plain |want|-relative rule"


DS = (256, 8, 7168, 2048)


@pytest.mark.parametrize("T,dt", [(1, "f16"), (1, "bf16"), (64, "f16"), (64, "bf16"), (8192, "f16"),
                                  (8192, "bf16")])
def test_deepseek_r1_layer(T, dt):
    got, want, scale, pick = _layer_case(*DS, T, dt, n_check=16, seed=100 + T, graph=(T == 64 and dt == "f16"))
    assert len(pick) == min(16, 8 * T)
    _check(got, want, scale, 0.99 if dt == "f16" else 0.9)


@pytest.mark.parametrize("dt", ["f16", "bf16"])
def test_deepseek_r1_decode_outliers(dt):
    """Heavy-tailed activations at K=7168 in decode mode: the offset codes carry a 1024*sum(x) term
    through the fp32 partials -- it must still cancel to within the bar."""
    got, want, scale, _ = _layer_case(*DS, 64, dt, n_check=16, seed=7, outliers=True)
    _check(got, want, scale, 0.99 if dt == "f16" else 0.9)


@pytest.mark.parametrize("T", [16, 2048])
def test_mixtral_layer(T):
    got, want, scale, _ = _layer_case(8, 2, 4096, 14336, T, "f16", n_check=8 if T == 16 else 3, seed=200 + T)
    _check(got, want, scale)


@pytest.mark.parametrize("zipf", [False, True])
def test_qwen3_layer(zipf):
    got, want, scale, _ = _layer_case(128, 8, 2048, 768, 256, "f16", n_check=16, seed=300, zipf=zipf)
    _check(got, want, scale)


def test_llama_dense_m4096():
    """Config 2 at its largest M: K=4096, N=14336, M=4096 (prefill tiles); 192 sampled rows checked."""
    from paper_2504_16214_b200.moe import w4a16_linear
    from paper_2504_16214_b200.moe.weights import random_packed
    M, N, K = 4096, 14336, 4096
    rng = np.random.default_rng(4096)
    w = random_packed(1, N, K, False, torch.float16, 77, "cuda")
    x = O.round_act(rng.standard_normal((M, K)).astype(np.float32) * 0.5, "f16")
    got = _from_dev_act(w4a16_linear(_to_dev_act(x, "f16"), w), "f16")
    rows = np.sort(np.concatenate([rng.choice(M, 160, replace=False), np.arange(M - 32, M)]))
    q, z, s = _expert_awq(77, 0, N, K, "f16")
    want = O.round_act(x[rows] @ O.dequant(q, z, s, "f16").T, "f16")
    np.testing.assert_allclose(got[rows], want, rtol=RTOL, atol=ATOL)


@pytest.mark.parametrize("ntok", [16, 128])
def test_grouped_gemm_rows_past_2_20(ntok):
    """More than 2^20 rows: the tile table's m_start keeps all 32 bits when there is no split-K (the
    20-bit field only exists for split-K launches, which need rows < 2^20)."""
    from paper_2504_16214_b200.moe import ops
    from paper_2504_16214_b200.moe.weights import random_packed
    E, N, K = 2, 128, 128
    counts = [(1 << 20) + 37, 91]
    rows = sum(counts)
    w = random_packed(E, N, K, False, torch.float16, 5, "cuda")
    g = torch.Generator(device="cuda").manual_seed(1)
    xd = (torch.randn((rows, K), generator=g, device="cuda") * 0.5).half()
    cnt = torch.tensor(counts, dtype=torch.int32, device="cuda")
    off = torch.tensor([0, counts[0], rows], dtype=torch.int32, device="cuda")
    xs = ops.group_sums(xd) if ntok == 16 else None
    out = ops.grouped_gemm(xd, w.blocks, E, N, False, cnt, off, ntok, xsum=xs)
    torch.cuda.synchronize()
    check = np.concatenate([np.arange(0, 64), np.arange(counts[0] - 200, rows)])
    x = xd[torch.from_numpy(check).cuda()].float().cpu().numpy()
    got = out[torch.from_numpy(check).cuda()].float().cpu().numpy()
    deq = [O.dequant(*_expert_awq(5, e, N, K, "f16"), "f16") for e in range(E)]
    want = np.stack([x[i] @ deq[0 if r < counts[0] else 1].T for i, r in enumerate(check)])
    np.testing.assert_allclose(got, O.round_act(want, "f16"), rtol=RTOL, atol=ATOL)
