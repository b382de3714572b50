"""The layout synthesizer and the sm_100a kernel agree on the int4 weight block.

Synthesizing the kernel's own tiles (tests/programs/sm100_{decode,prefill}_tile.prog) against the B200
catalog (tilesynth/data/sm100.cat: tcgen05 MMA with the weight operand in tensor memory) must give:

* the register layout the kernel uses for dequantisation -- one weight row per thread of the 4-warp
  dequant group (TMEM lane = row), the k values of the row as that thread's values;
* the per-iteration block order derived from it (tilesynth.repack.block_order, the SURVEY Appendix-A
  repack recipe with one 16-byte vector per iteration) == the shared buffer the synthesizer
  materialises == csrc/w4_format.cuh's packed block: element (n, k) at (k / 32) * 4096 + n * 32 + k % 32,
  copied with 16 B vectors both ways, conflict-free without a swizzle, and servable by the bulk
  tensor engine (check_tma);
* and (GPU) the bytes w4a16_repack_awq writes place every (n, k) exactly there -- up to the
  documented nibble interleave inside each 32-bit word (slot_of(e) = (e & 1) * 4 + (e >> 1), the
  dequantiser's LOP3 pairing, which the synthesizer does not model: it works in whole elements).
"""
from pathlib import Path

import numpy as np
import pytest

from paper_2504_16214_b200.tilesynth import algebra as A
from paper_2504_16214_b200.tilesynth import explore as X
from paper_2504_16214_b200.tilesynth import isa_table as C
from paper_2504_16214_b200.tilesynth import tileprog as P
from paper_2504_16214_b200.tilesynth.layout_flow import SynthesisConfig
from paper_2504_16214_b200.tilesynth.repack import block_order, tma_plan

PROGS = Path(__file__).resolve().parent / "programs"
KERNEL_BLOCK = "(128,(32,4)):(32,(1,4096))"  # csrc/w4_format.cuh, in int4 elements


def _kernel_offset(n, k):
    return (k // 32) * 4096 + n * 32 + k % 32


def _synth(name):
    cat = C.load_catalog(C.builtin_catalog_path("sm100"))
    g = P.parse_program((PROGS / name).read_text())
    res = X.synthesize_program(g, cat, SynthesisConfig(threads=128, max_candidates=64))
    assert res.ok, res.diagnostics
    return res


@pytest.mark.parametrize("prog", ["sm100_decode_tile.prog", "sm100_prefill_tile.prog"])
def test_synthesized_weight_block_is_the_kernel_block(prog):
    res = _synth(prog)
    best = res.best
    w4 = best.layouts["w4"]
    # one row per thread (TMEM lane = row), the row's 128 k values per thread
    t_mode, v_mode = A.coalesce(w4.layout.mode(0)), A.coalesce(w4.layout.mode(1))
    assert (str(t_mode), str(v_mode)) == ("(128):(1)", "(128):(128)")
    order = block_order(w4, 32, (128, 128))  # 32 int4 = one 16-byte vector per thread and iteration
    assert str(order) == KERNEL_BLOCK
    assert all(order((n, k)) == _kernel_offset(n, k) for n in range(0, 128, 7) for k in range(128))
    # the materialised shared buffer is the same order, conflict-free with the identity swizzle
    sw = best.smem["sw"]
    assert str(sw.layout) == KERNEL_BLOCK and sw.swizzle.is_identity
    assert set(sw.copy_conflicts.values()) == {1}
    copies = {op.index: best.choices[op.index].name for op in res.graph.ops if op.kind == "copy"}
    assert copies[2] == "cp_async_128" and copies[3] == "lds_128"  # 16 B both ways
    # the bulk tensor engine can fill it (what the kernel does: one bulk copy per block)
    plan = tma_plan(res)
    assert plan["sw"]["feasible"] and plan["sw"]["hint"] == KERNEL_BLOCK


def test_appendix_a_thread_major_recipe_is_the_one_vector_case():
    """vector_elems = V reproduces the SURVEY recipe (thread-major: a row per thread, contiguous)."""
    w4 = _synth("sm100_decode_tile.prog").best.layouts["w4"]
    assert str(block_order(w4, 128, (128, 128))) == "(128,128):(128,1)"


def test_awq_native_order_is_not_synthesizable():
    """The AWQ checkpoint order of the same tile (k-major, 8 codes per int32 along n) finds no
    16 B plan (the reference's observation for its AWQ-native program)."""
    text = (PROGS / "sm100_decode_tile.prog").read_text().replace(
        "bufW int4 (128,(32,4)):(32,(1,4096))", "bufW int4 (((2,4),16),128):(((4,1),8),128)")
    cat = C.load_catalog(C.builtin_catalog_path("sm100"))
    res = X.synthesize_program(P.parse_program(text), cat, SynthesisConfig(threads=128, max_candidates=64))
    if res.ok:  # a plan exists only with narrow copies
        widths = {res.best.choices[op.index].vector_bytes for op in res.graph.ops
                  if op.kind == "copy" and op.index in res.best.choices and "sw" in op.operands + op.results}
        assert max(widths) < 16
    else:
        assert res.diagnostics


@pytest.mark.gpu
def test_kernel_repack_bytes_follow_the_synthesized_order():
    """Probe w4a16_repack_awq with codes that spell out their own (n, k) (4 bit planes of n*128+k)
    and read back where each element landed."""
    import torch
    import moe_oracle as O
    from paper_2504_16214_b200.moe import ops
    N = K = 128
    idx = (np.arange(N)[:, None] * K + np.arange(K)[None, :]).astype(np.int64)
    seen = np.zeros(N * K, dtype=np.int64)
    z = np.zeros((1, N, K // 128), np.uint8)
    s = np.ones((1, N, K // 128), np.float32)
    for plane in range(4):
        q = ((idx >> (4 * plane)) & 15).astype(np.uint8)[None]
        qw, sc, qz = O.to_awq(q, z, s)
        blocks = ops.repack_awq(torch.from_numpy(qw).cuda(), torch.from_numpy(sc).cuda().half(),
                                torch.from_numpy(qz).cuda(), parts=1)
        codes = blocks[:8192].cpu().numpy()
        nib = np.stack([codes & 15, codes >> 4], axis=1).reshape(-1).astype(np.int64)  # physical nibble order
        seen |= nib << (4 * plane)
    # physical nibble i of a 32-bit word holds element e with slot_of(e) = i
    slot_of = np.array([(e & 1) * 4 + (e >> 1) for e in range(8)])
    logical = np.empty_like(seen)
    words = seen.reshape(-1, 8)
    logical.reshape(-1, 8)[:, np.arange(8)] = words[:, slot_of]
    w4 = _synth("sm100_decode_tile.prog").best.layouts["w4"]
    order = block_order(w4, 32, (N, K))
    want = np.empty(N * K, dtype=np.int64)
    for n in range(N):
        for k in range(K):
            want[order((n, k))] = n * K + k
    assert np.array_equal(logical, want)
