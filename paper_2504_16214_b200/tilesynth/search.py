"""Candidate search: one leaf per assignment of copy instructions, in lexicographic order of the
per-copy option lists (widest first), up to the candidate cap; the all-narrowest assignment is
always tried last. A leaf = TV propagation over every component + shared-buffer synthesis +
staging buffers for redistributions; leaves that fail with a pruning error are dropped.

Leaf semantics and order are the reference's (``/root/reference/pkg/src/tilesynth/synth.py``:
``_copy_choice_points`` ``:533``, ``evaluate_assignment`` ``:547-563``, shared / staging synthesis
``:566-662``, ``expand_search`` ``:665-720``). Unlike a plain DFS, the walk here memoises
propagation per register-connected component: a component's layouts depend only on the
instructions chosen for its own copies, so the leaves of a search tree share (and, when a
component fails, prune on) each component outcome instead of recomputing it.
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

from .errors import (LayoutIncompatible, NoInstructionAvailable, NonDivisibleTile, NotDivisible, NotInvertible,
                     OutOfDomain, ShapeMismatch, StrideConflict, Unsatisfiable)
from .instr_catalog import Catalog, Instruction, candidates_for_copy
from .smem_layout import BufferCopy, SmemLayout, synthesize_buffer
from .tile_ir import OpNode, ProgramGraph, TensorDecl, partition_components
from .tv_solver import PropagationState, RearrangePatch, SlotKey, SynthesisConfig, propagate
from .tvl import TvLayout

# failures that only disqualify one leaf (anything else aborts the search)
PRUNE = (LayoutIncompatible, NonDivisibleTile, NotDivisible, NotInvertible, OutOfDomain, ShapeMismatch,
         StrideConflict, Unsatisfiable, NoInstructionAvailable)
_PRUNE_ERRORS = PRUNE


@dataclass
class Candidate:
    index: int
    choices: Dict[int, Instruction]
    layouts: Dict[SlotKey, TvLayout]
    patches: List[RearrangePatch]
    smem: Dict[str, SmemLayout]
    staging: Dict[str, SmemLayout] = field(default_factory=dict)
    cost: Optional[object] = None


def _copy_choice_points(graph: ProgramGraph, catalog: Catalog) -> List[Tuple[OpNode, List[Instruction]]]:
    """(copy op, its options widest first) for every copy that needs an instruction."""
    out = []
    for op in graph.ops:
        if op.kind == "copy":
            src, dst = graph.tensor(op.operands[0]), graph.tensor(op.results[0])
            if not (src.scope == dst.scope == "Register"):
                out.append((op, candidates_for_copy(catalog, src, dst)))
    return out


class _View:
    """The slice of PropagationState the buffer passes read."""

    def __init__(self, layouts, patches):
        self.layouts, self.patches = layouts, patches


def _component_outcome(component, graph, catalog, config, picked: Dict[int, Instruction]):
    """Propagate one component on its own state -> (layouts, patches, matrix instructions)."""
    state = PropagationState(graph, config)
    local = dict(picked)
    propagate(component, graph, local, config, catalog, state)
    extra = {k: v for k, v in local.items() if k not in picked}
    return state.layouts, state.patches, extra


def _shared_buffers(graph: ProgramGraph, choices: Dict[int, Instruction], layouts) -> Dict[str, SmemLayout]:
    users: Dict[str, List[BufferCopy]] = {}
    for op in graph.ops:
        if op.kind != "copy":
            continue
        for name, side in ((op.operands[0], "src"), (op.results[0], "dst")):
            decl = graph.tensor(name)
            if decl.scope == "Shared":
                inst = choices[op.index]
                users.setdefault(name, []).append(
                    BufferCopy(op.index, layouts[(op.index, side)], inst.vector_elems(decl.dtype), inst.name))
    return {name: synthesize_buffer(name, graph.tensor(name).shape, graph.tensor(name).dtype.bits, users[name])
            for name in sorted(users)}


def _synthesize_shared(graph: ProgramGraph, choices: Dict[int, Instruction], state) -> Dict[str, SmemLayout]:
    return _shared_buffers(graph, choices, state.layouts)


def _staging_instructions(catalog: Catalog, decl: TensorDecl) -> List[Tuple[Instruction, Instruction]]:
    """(store, load) pairs of equal width for a round trip through a staging buffer, widest first
    (loads: the first generic one of each width)."""
    staging = TensorDecl("staging", "Shared", decl.dtype, decl.shape)
    loads: Dict[int, Instruction] = {}
    for inst in candidates_for_copy(catalog, staging, decl):
        if inst.generic:
            loads.setdefault(inst.vector_bytes, inst)
    return [(st, loads[st.vector_bytes]) for st in candidates_for_copy(catalog, decl, staging)
            if st.vector_bytes in loads]


def _synthesize_staging(graph: ProgramGraph, catalog: Catalog, config: SynthesisConfig, state) -> Dict[str, SmemLayout]:
    """Staging buffers for user rearranges and inserted redistributions (first workable pair)."""
    layouts = state.layouts
    jobs = [(f"rearrange@{op.index}", op.operands[0], layouts[op.operands[0]], layouts[op.results[0]])
            for op in graph.ops
            if op.kind == "rearrange" and op.operands[0] in layouts and op.results[0] in layouts]
    jobs += [(f"redistribute@{p.op_index}:{p.tensor}", p.tensor, p.from_layout, p.to_layout) for p in state.patches]
    out: Dict[str, SmemLayout] = {}
    for label, tensor, src_tv, dst_tv in jobs:
        decl = graph.tensor(tensor)
        for store, load in _staging_instructions(catalog, decl):
            copies = [BufferCopy(-1, src_tv, store.vector_elems(decl.dtype), store.name),
                      BufferCopy(-2, dst_tv, load.vector_elems(decl.dtype), load.name)]
            try:
                out[label] = synthesize_buffer(label, decl.shape, decl.dtype.bits, copies)
                break
            except PRUNE:
                continue
        else:
            raise Unsatisfiable(f"no staging layout for redistribution of {tensor}")
    return out


class _Leaves:
    """Evaluates leaves of one search, caching component outcomes (or their failures)."""

    def __init__(self, graph: ProgramGraph, catalog: Catalog, config: SynthesisConfig):
        self.graph, self.catalog, self.config = graph, catalog, config
        self.components = partition_components(graph)
        self.copy_ops = [[op.index for op in comp if op.kind == "copy"] for comp in self.components]
        self.memo: Dict[Tuple, object] = {}

    def component(self, i: int, picked: Dict[int, Instruction]):
        mine = {k: picked[k] for k in self.copy_ops[i] if k in picked}
        key = (i, tuple(sorted((k, v.name) for k, v in mine.items())))
        hit = self.memo.get(key)
        if hit is None:
            try:
                hit = _component_outcome(self.components[i], self.graph, self.catalog, self.config, mine)
            except Exception as e:  # noqa: BLE001 -- replayed verbatim for every leaf sharing it
                hit = e
            self.memo[key] = hit
        if isinstance(hit, Exception):
            raise hit
        return hit

    def evaluate(self, picked: Dict[int, Instruction]):
        choices = dict(picked)
        layouts: Dict[SlotKey, TvLayout] = {}
        patches: List[RearrangePatch] = []
        for i in range(len(self.components)):
            got_layouts, got_patches, mma = self.component(i, picked)
            layouts.update(got_layouts)
            patches.extend(got_patches)
            choices.update(mma)
        view = _View(layouts, patches)
        smem = _shared_buffers(self.graph, choices, layouts)
        staging = _synthesize_staging(self.graph, self.catalog, self.config, view)
        return choices, layouts, patches, smem, staging


def evaluate_assignment(graph: ProgramGraph, catalog: Catalog, config: SynthesisConfig,
                        choices: Dict[int, Instruction]):
    """One leaf: (completed choices, layouts, patches, shared buffers, staging buffers)."""
    state = PropagationState(graph, config)
    for component in partition_components(graph):
        propagate(component, graph, choices, config, catalog, state)
    return (choices, state.layouts, state.patches, _synthesize_shared(graph, choices, state),
            _synthesize_staging(graph, catalog, config, state))


def expand_search(graph: ProgramGraph, catalog: Catalog, config: SynthesisConfig) -> List[Candidate]:
    """Valid leaves in lexicographic option order, capped at ``max_candidates - 1`` (the last slot
    is kept for the all-narrowest leaf, evaluated if not already found); ``Candidate.index`` is the
    discovery order."""
    if not graph.ops:
        return []
    points = _copy_choice_points(graph, catalog)
    leaves = _Leaves(graph, catalog, config)
    found: List[Candidate] = []
    valid_keys = set()
    cap = max(1, config.max_candidates - 1)

    def visit(key: Tuple[int, ...]) -> Optional[Candidate]:
        picked = {op.index: options[i] for (op, options), i in zip(points, key)}
        try:
            result = leaves.evaluate(picked)
        except PRUNE:
            return None
        return Candidate(len(found), *result)

    for key in itertools.product(*(range(len(options)) for _, options in points)):
        if len(found) >= cap:
            break
        cand = visit(key)
        if cand is not None:
            found.append(cand)
            valid_keys.add(key)
    narrowest = tuple(len(options) - 1 for _, options in points)
    if config.max_candidates > 1 and narrowest not in valid_keys:
        cand = visit(narrowest)
        if cand is not None:
            found.append(cand)
    return found
