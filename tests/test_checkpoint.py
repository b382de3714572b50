"""AWQ checkpoint loading (safetensors, HuggingFace per-expert naming) and the packed on-disk format;
the vLLM-style FusedMoE method on a plain module. CPU tests: container round trip and stacking, bit
exact against the oracle's AWQ packing; GPU tests: load -> repack -> layer == the oracle layer."""
import numpy as np
import pytest
import torch

import moe_oracle as O
from paper_2504_16214_b200.moe import checkpoint as ck

E, H, I, G = 4, 256, 128, 128


def _layer_awq(rng, dt="f16"):
    """HF-style per-expert AWQ tensors of one MoE layer + the logical (q, z, s) they encode."""
    tdt = torch.float16 if dt == "f16" else torch.bfloat16
    q13, z13, s13 = O.synth_awq_expert_weights(rng, E, 2 * I, H, dt)
    q2, z2, s2 = O.synth_awq_expert_weights(rng, E, H, I, dt)
    tensors = {}
    for e in range(E):
        for proj, (q, z, s) in (("gate_proj", (q13[e, :I], z13[e, :I], s13[e, :I])),
                                ("up_proj", (q13[e, I:], z13[e, I:], s13[e, I:])),
                                ("down_proj", (q2[e], z2[e], s2[e]))):
            qw, sc, qz = O.to_awq(q[None], z[None], s[None])
            tensors[f"model.layers.3.mlp.experts.{e}.{proj}.qweight"] = torch.from_numpy(qw[0])
            tensors[f"model.layers.3.mlp.experts.{e}.{proj}.qzeros"] = torch.from_numpy(qz[0])
            tensors[f"model.layers.3.mlp.experts.{e}.{proj}.scales"] = torch.from_numpy(sc[0]).to(tdt)
    return tensors, (q13, z13, s13, q2, z2, s2)


def test_safetensors_round_trip(tmp_path):
    rng = np.random.default_rng(0)
    tensors, _ = _layer_awq(rng, "bf16")
    tensors["empty"] = torch.empty((0, 3), dtype=torch.float32)
    p = tmp_path / "layer.safetensors"
    ck.write_safetensors(p, tensors, {"note": "fixture"})
    back, meta = ck.read_safetensors(p)
    assert meta == {"note": "fixture"} and set(back) == set(tensors)
    for k, v in tensors.items():
        assert back[k].dtype == v.dtype and back[k].shape == v.shape
        assert torch.equal(back[k].view(torch.uint8) if v.numel() else back[k], v.view(torch.uint8) if v.numel() else v)
    raw = p.read_bytes()  # container layout: u64 header length, JSON header, 8-byte aligned payload
    n = int.from_bytes(raw[:8], "little")
    assert (8 + n) % 8 == 0 and raw[8:9] == b"{"


def test_stack_matches_vllm_layout():
    """Per-expert gate/up/down -> w13 = [gate | up] along N, stacked over experts: exactly the oracle's
    AWQ packing of the full w13 / w2 (vLLM's AWQ MoE parameter layout)."""
    rng = np.random.default_rng(1)
    tensors, (q13, z13, s13, q2, z2, s2) = _layer_awq(rng)
    st = ck.stack_awq_experts(tensors, "model.layers.3.mlp.experts", E)
    for name, (q, z, s) in (("w13", (q13, z13, s13)), ("w2", (q2, z2, s2))):
        qw, sc, qz = O.to_awq(q, z, s)
        assert np.array_equal(st[f"{name}_qweight"].numpy(), qw)
        assert np.array_equal(st[f"{name}_qzeros"].numpy(), qz)
        assert np.array_equal(st[f"{name}_scales"].float().numpy(), sc)
    with pytest.raises(KeyError, match="experts.4"):
        ck.stack_awq_experts(tensors, "model.layers.3.mlp.experts", E + 1)


@pytest.mark.gpu
def test_load_pack_save_layer(tmp_path):
    from paper_2504_16214_b200.moe import moe_w4a16
    rng = np.random.default_rng(2)
    tensors, (q13, z13, s13, q2, z2, s2) = _layer_awq(rng)
    p = tmp_path / "layer.safetensors"
    ck.write_safetensors(p, tensors)
    w = ck.load_awq_moe(p, "model.layers.3.mlp.experts", E)
    T, k = 20, 2
    x = O.round_act(rng.standard_normal((T, H)).astype(np.float32) * 0.5, "f16")
    ids, wts = O.route_topk(rng.standard_normal((T, E)).astype(np.float32), k, "softmax", True)
    xd = torch.from_numpy(x).cuda().half()
    idd, wd = torch.from_numpy(ids).cuda(), torch.from_numpy(wts).cuda()
    y = moe_w4a16(xd, w, wd, idd)
    want = O.moe_forward(x, O.dequant(q13, z13, s13, "f16"), O.dequant(q2, z2, s2, "f16"), ids, wts, "f16")
    np.testing.assert_allclose(y.float().cpu().numpy(), want, rtol=1e-2, atol=1e-2)
    pk = tmp_path / "layer.w4a16.safetensors"
    ck.save_packed(pk, w)
    w2 = ck.load_packed(pk)
    assert torch.equal(w2.w13.blocks, w.w13.blocks) and torch.equal(w2.w2.blocks, w.w2.blocks)
    assert (w2.num_experts, w2.hidden, w2.inter, w2.w13.dtype) == (E, H, I, torch.float16)
    assert torch.equal(moe_w4a16(xd, w2, wd, idd), y)


@pytest.mark.gpu
def test_vllm_style_method_on_module():
    """create_weights -> (loader fills the AWQ params) -> process_weights_after_loading -> apply."""
    from paper_2504_16214_b200.moe.vllm_method import W4A16MoEMethod
    rng = np.random.default_rng(3)
    tensors, (q13, z13, s13, q2, z2, s2) = _layer_awq(rng)
    st = ck.stack_awq_experts(tensors, "model.layers.3.mlp.experts", E)
    layer = torch.nn.Module()
    m = W4A16MoEMethod()
    m.create_weights(layer, E, H, I, torch.float16, weight_loader=None)
    for name, t in st.items():
        getattr(layer, name).data = t.cuda()
    m.process_weights_after_loading(layer)
    assert layer.w13_qweight.numel() == 0  # AWQ copies released after the repack
    T, k = 9, 2
    x = O.round_act(rng.standard_normal((T, H)).astype(np.float32) * 0.5, "f16")
    lg = rng.standard_normal((T, E)).astype(np.float32)
    xd = torch.from_numpy(x).cuda().half()
    y_logits = m.apply(layer, xd, router_logits=torch.from_numpy(lg).cuda(), top_k=k, renormalize=True)
    ids, wts = O.route_topk(lg, k, "softmax", True)
    y_routed = m.apply(layer, xd, torch.from_numpy(wts).cuda(), torch.from_numpy(ids).cuda())
    want = O.moe_forward(x, O.dequant(q13, z13, s13, "f16"), O.dequant(q2, z2, s2, "f16"), ids, wts, "f16")
    for y in (y_logits, y_routed):
        np.testing.assert_allclose(y.float().cpu().numpy(), want, rtol=1e-2, atol=1e-2)
