"""CPU tests of the numeric oracle itself (oracle/moe_oracle.py): pinned against vLLM's AWQ packing
golden vectors and against independent restatements of the rounding/routing/permutation rules."""
from pathlib import Path

import numpy as np
import pytest

import moe_oracle as O

GOLD = Path(__file__).resolve().parent / "golden" / "awq_pack_vllm.npz"


@pytest.mark.parametrize("shape", ["8x8", "16x64", "128x256"])
def test_awq_pack_matches_vllm(shape):
    g = np.load(GOLD)
    q, packed = g[f"q_{shape}"], g[f"packed_{shape}"]
    assert np.array_equal(O.awq_pack(q), packed)
    assert np.array_equal(O.awq_unpack(packed), q)


def test_awq_unpack_is_vllm_reverse_order():
    # column c of a packed word sits at nibble slot [0,4,1,5,2,6,3,7][c] (vllm awq_marlin.py:70-74)
    q = np.arange(8, dtype=np.uint8)[None, :]
    w = int(O.awq_pack(q).view(np.uint32)[0, 0])
    slots = [(w >> (4 * s)) & 15 for s in range(8)]
    assert slots == [0, 2, 4, 6, 1, 3, 5, 7]


@pytest.mark.parametrize("dt", ["f16", "bf16"])
def test_dequant_single_rounding(dt):
    rng = np.random.default_rng(3)
    q = rng.integers(0, 16, size=(4, 256), dtype=np.uint8)
    z = rng.integers(0, 16, size=(4, 2), dtype=np.uint8)
    s = O.round_act(rng.uniform(-2, 2, size=(4, 2)).astype(np.float32), dt)
    w = O.dequant(q, z, s, dt)
    # exact product in float64, one rounding to the act dtype
    exact = (q.astype(np.float64) - np.repeat(z, 128, 1)) * np.repeat(s.astype(np.float64), 128, 1)
    assert np.array_equal(w, O.round_act(exact.astype(np.float32), dt))
    assert np.array_equal(O.act_bits(w, dt), O.act_bits(O.round_act(w, dt), dt))


def test_round_bf16_ties_to_even():
    x = np.array([1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, -(1.0 + 2 ** -8), 65504.0], np.float32)
    r = O.round_bf16(x)
    assert r[0] == 1.0 and r[1] == 1.0 + 2 ** -6 and r[2] == -1.0


def test_route_topk_ties_and_weights():
    lg = np.zeros((2, 6), np.float32)
    lg[1] = [0.5, 2.0, 2.0, -1.0, 2.0, 0.0]
    ids, w = O.route_topk(lg, 3, "softmax", renormalize=False)
    assert ids.tolist() == [[0, 1, 2], [1, 2, 4]]
    assert np.allclose(w[0], 1 / 6)
    ids, w = O.route_topk(lg, 2, "sigmoid", renormalize=True)
    assert ids[1].tolist() == [1, 2] and np.allclose(w.sum(1), 1.0)


def test_permute_is_stable_counting_sort():
    rng = np.random.default_rng(0)
    ids = rng.integers(-1, 9, size=(50, 4)).astype(np.int32)
    counts, offsets, sp, pp = O.moe_permute(ids, 8)
    flat = ids.reshape(-1)
    valid = np.nonzero((flat >= 0) & (flat < 8))[0]
    expect = sorted(valid.tolist(), key=lambda i: (flat[i], i))
    assert sp.tolist() == expect
    assert counts.tolist() == [int((flat == e).sum()) for e in range(8)]
    assert all(pp[i] == -1 for i in range(flat.size) if i not in set(valid.tolist()))
    assert all(sp[pp[i]] == i for i in valid)


def test_moe_forward_linearity_in_routing_weights():
    rng = np.random.default_rng(1)
    T, E, k, H, I = 5, 4, 2, 128, 128
    q13, z13, s13 = O.synth_awq_expert_weights(rng, E, 2 * I, H, "f16")
    q2, z2, s2 = O.synth_awq_expert_weights(rng, E, H, I, "f16")
    x = O.round_act(rng.standard_normal((T, H)).astype(np.float32), "f16")
    ids = np.stack([rng.permutation(E)[:k] for _ in range(T)]).astype(np.int32)
    w = np.full((T, k), 0.5, np.float32)
    y = O.moe_forward(x, O.dequant(q13, z13, s13, "f16"), O.dequant(q2, z2, s2, "f16"), ids, w, "f16")
    y2 = O.moe_forward_expertwise(x, q13, z13, s13, q2, z2, s2, ids, w, "f16")
    assert np.array_equal(y, y2)


def test_group_sums_restatement():
    """(C, S) group sums: direct loop vs the vectorised restatement, both dtypes."""
    rng = np.random.default_rng(3)
    x = O.round_act(rng.standard_normal((5, 256)).astype(np.float32), "f16")
    for dt in ("f16", "bf16"):
        got = O.group_sums(x, dt)
        assert got.shape == (2, 5, 2)
        for g in range(2):
            for r in range(5):
                xs = x[r, g * 128:(g + 1) * 128].astype(np.float64)
                c = np.array([128.0 if dt == "bf16" else (64.0 if (k % 8) in (2, 3, 6, 7) else 1024.0)
                              for k in range(128)])
                assert np.isclose(got[g, r, 1], xs.sum(), rtol=1e-6, atol=1e-4)
                assert np.isclose(got[g, r, 0], (c * xs).sum(), rtol=1e-6, atol=1e-2)


GOLD_GT = Path(__file__).resolve().parent / "golden" / "grouped_topk_vllm.npz"


@pytest.mark.parametrize("case", ["ds_r1", "ds_r1_nobias", "softmax_g4", "softmax_bias"])
def test_grouped_topk_matches_vllm(case):
    """The grouped top-k restatement == vLLM 0.22's torch grouped_topk on the golden vectors
    (tools/make_golden_grouped_topk.py; slots ordered by descending weight)."""
    g = np.load(GOLD_GT)
    T, E, k, G, TG, softmax, renorm, use_bias = (int(v) for v in g[f"{case}_meta"])
    bias = g[f"{case}_bias"] if use_bias else None
    ids, w = O.grouped_topk(g[f"{case}_logits"], k, G, TG, "softmax" if softmax else "sigmoid", bool(renorm), bias,
                            float(g[f"{case}_scale"][0]))
    order = np.argsort(-w, axis=1, kind="stable")
    np.testing.assert_array_equal(np.take_along_axis(ids, order, axis=1), g[f"{case}_ids"])
    np.testing.assert_allclose(np.take_along_axis(w, order, axis=1), g[f"{case}_weights"], rtol=1e-6, atol=1e-7)


def test_grouped_topk_group_rule():
    """Experts outside the kept groups are never chosen, even when their scores are the largest."""
    lg = np.full((1, 16), -3.0, dtype=np.float32)
    lg[0, 0] = 5.0                  # group 0 (experts 0-3): one huge expert, the rest small
    lg[0, 4:8] = 1.0                # group 1: uniformly medium (bias-free group score = max = 1 < 5)
    lg[0, 8:12] = [2.0, 2.0, -9, -9]
    ids, _ = O.grouped_topk(lg, 2, 4, 1, "sigmoid", True, None)
    assert set(ids[0].tolist()) <= {0, 1, 2, 3}
    bias = np.zeros(16, dtype=np.float32)  # with a bias the group score is the sum of the best two
    ids, _ = O.grouped_topk(lg, 2, 4, 1, "sigmoid", True, bias)
    assert set(ids[0].tolist()) <= {8, 9, 10, 11}


GOLD_VLLM = Path(__file__).resolve().parent / "golden" / "vllm_moe.npz"  # tools/make_golden_vllm.py (GPU)


@pytest.mark.parametrize("case", range(6))
def test_route_topk_matches_vllm_kernel(case):
    """Softmax / sigmoid top-k == vLLM 0.22's CUDA topk_softmax / topk_sigmoid (the fused_topk of its
    FusedMoE): ids bit-exact (ties and an all-equal row included), weights to fp32 rounding."""
    d = np.load(GOLD_VLLM)
    T, E, k, soft, rn = (int(v) for v in d[f"route{case}_meta"])
    ids, w = O.route_topk(d[f"route{case}_logits"], k, "softmax" if soft else "sigmoid", bool(rn))
    assert np.array_equal(ids, d[f"route{case}_ids"])
    np.testing.assert_allclose(w, d[f"route{case}_w"], rtol=2e-6, atol=2e-7)


@pytest.mark.parametrize("layer", range(2))
def test_moe_forward_matches_vllm_w4a16_moe(layer):
    """The oracle's W4A16 MoE layer (dequant to the activation dtype, SwiGLU, h and the expert outputs
    rounded to it, fp32 combine) == vLLM 0.22's fused_experts with int4_w4a16 (its moe_wna16 Triton
    path for AWQ) on the same weights and routing, within rtol / atol 1e-2 (fp16 and bf16)."""
    d = np.load(GOLD_VLLM)
    T, E, k, H, I, f16 = (int(v) for v in d[f"layer{layer}_meta"])
    g = lambda n: d[f"layer{layer}_{n}"]  # noqa: E731
    want = O.moe_forward_expertwise(g("x"), g("q13"), g("z13"), g("s13"), g("q2"), g("z2"), g("s2"), g("ids"),
                                    g("w"), "f16" if f16 else "bf16")
    np.testing.assert_allclose(want, g("y"), rtol=1e-2, atol=1e-2)
