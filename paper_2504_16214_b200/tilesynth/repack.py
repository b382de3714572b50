"""From a synthesized register layout to the global block order of a weight operand, and the TMA
plan of shared buffers -- the link between the layout synthesizer and the sm_100a kernels.

SURVEY.md Appendix A gives the reference-side recipe: take the synthesized int4 register layout
``f`` of the weight tile, ``fr = filter_replication(f)`` (tv.py:140), and store element p of the tile
at ``t * V + v`` where ``(t, v) = inverse(fr)(p)`` (layout.py:302): each thread's values become one
contiguous run, regrouped by the tile extents (layout.py:415). :func:`block_order` generalises the
run to one copy *iteration*: with a ``vector_elems``-element vector per thread and instruction, the
T threads' vectors of iteration j are stored next to each other,

    offset(t, v) = (v // vec) * (T * vec) + t * vec + v % vec,

so every warp-wide vector load reads one contiguous span (conflict-free without a swizzle) and a
bulk copy of the block lands in shared memory already in that order. ``vector_elems = V`` is the
Appendix-A recipe itself.

For the decode tile of ``csrc/w4a16_gemm.cu`` synthesized against ``data/sm100.cat`` (tcgen05 MMA
with the weight operand in tensor memory: one row per thread of the 4-warp dequant group) this
yields ``(128,(32,4)):(32,(1,4096))`` -- exactly the packed block format of ``csrc/w4_format.cuh``
(chunk-major, 128 rows x 16 B per 32-k chunk). tests/test_synth_kernel_link.py checks it against the
synthesizer and against the bytes ``w4a16_repack_awq`` writes.
"""
from __future__ import annotations

from .algebra import Layout, coalesce, compose, group_modes, inverse
from .isa_table import tma_candidates
from .smem_plan import check_tma
from .algebra import filter_replication


def block_order(tv, vector_elems, extents):
    """Global (extents) -> storage offset layout that stores ``tv``'s per-thread vectors iteration
    by iteration (see the module docstring). ``tv`` may carry broadcast digits (dropped first)."""
    fr = filter_replication(tv)
    T, V = fr.threads, fr.values
    if V % vector_elems:
        raise ValueError(f"{V} values per thread do not split into {vector_elems}-element vectors")
    per_iteration = Layout((T, (vector_elems, V // vector_elems)), (vector_elems, (1, T * vector_elems)))
    return group_modes(coalesce(compose(per_iteration, inverse(fr.layout))), tuple(extents))


def tma_plan(result):
    """Per shared buffer of the best candidate: can the catalog's bulk tensor engine serve it?
    {buffer: {instruction, feasible, reason, hint}} for the buffers a TMA-flagged instruction could
    fill or drain (none for catalogs without TMA entries, e.g. sm80)."""
    cand, graph, cat = result.best, result.graph, result.catalog
    if cand is None:
        return {}
    plan = {}
    for name, smem in sorted(cand.smem.items()):
        decl = graph.tensor(name)
        engines = []
        for op in graph.ops:
            if op.kind == "copy" and name in (op.operands[0], op.results[0]):
                engines += tma_candidates(cat, graph.tensor(op.operands[0]), graph.tensor(op.results[0]))
        if not engines or smem.constraint is None:
            continue
        chk = check_tma(smem.constraint, decl.dtype.bits, max_dims=cat.tma_max_dims, align_bytes=cat.tma_align_bytes,
                        max_box=cat.tma_max_box)
        plan[name] = {"instruction": engines[0].name, "feasible": chk.feasible, "reason": chk.reason,
                      "hint": str(chk.hint) if chk.hint is not None else None}
    return plan
