"""Thread-value layout inference over one register-connected component (paper Algorithm 1).

Anchors fix the first layouts -- matrix ops by tiling their output with the instruction fragments
(warps along rows first), otherwise the largest global copy by address-ordered coalescing. Then
constraints are discharged in *rounds*: every round takes the constraints with at most one unknown
slot at the start of the round and solves them in list order; a demand that contradicts a layout
already assigned becomes a redistribution patch on the solving op instead of an error.

Semantics (solutions, patch placement, diagnostics text) are the reference's
(``/root/reference/pkg/src/tilesynth/synth.py``: anchors ``:125-256``, ``solve_copy`` ``:262-293``,
constraints ``:313-357``, state ``:360-386``, ``propagate`` ``:416-480``). The anchor and copy
solutions are pure functions of immutable inputs and are memoised, because the candidate search
re-derives the same ones for most of its leaves.
"""
from __future__ import annotations

import functools
import math
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Tuple, Union

from .errors import (LayoutIncompatible, NoInstructionAvailable, NonDivisibleTile, NotDivisible, NotInvertible,
                     OutOfDomain, ShapeMismatch, UnsolvedResidual)
from .instr_catalog import Catalog, Instruction, fastest_mma
from .layout_algebra import Layout, compose, inverse
from .tile_ir import DType, OpNode, ProgramGraph, TensorDecl
from .tvl import TvLayout, restrict_tv, tv_from_mode_lists

SlotKey = Union[str, Tuple[int, str]]


@dataclass
class SynthesisConfig:
    threads: int = 128
    max_candidates: int = 64

    def __post_init__(self):
        if self.threads < 32 or self.threads % 32:
            raise ValueError("thread count must be a positive multiple of 32")

    @property
    def warps(self) -> int:
        return self.threads // 32


@dataclass
class RearrangePatch:
    """A register redistribution: ``op_index`` reads / writes ``tensor`` as ``to_layout`` while the
    tensor itself keeps ``from_layout``."""

    op_index: int
    tensor: str
    from_layout: TvLayout
    to_layout: TvLayout
    inserted: bool = True   # False for user-written rearrange ops


@dataclass
class TvConstraint:
    kind: str               # "copy" | "elem" | "reduce" | "gemm_rows" | "gemm_cols" | "gemm_red"
    op: OpNode
    slots: List[SlotKey]
    tensors: List[str]
    solved: bool = False


def slot_for(graph: ProgramGraph, op: OpNode, tensor: str) -> SlotKey:
    """Register tensors have one layout program-wide; a Global / Shared operand gets a per-op side."""
    if graph.tensor(tensor).scope == "Register":
        return tensor
    if op.kind == "copy":
        return op.index, ("src" if tensor == op.operands[0] else "dst")
    return op.index, ("src" if tensor in op.operands else "dst")


def _runs(layout: Layout, mode: int) -> List[Tuple[int, int]]:
    return layout.mode(mode).flat_modes()


def _colex_weights(extents: Sequence[int]) -> Tuple[int, ...]:
    return tuple(math.prod(extents[:i]) for i in range(len(extents)))


# ------------------------------------------------------------------------------------------ anchors
@functools.lru_cache(maxsize=4096)
def _coalesced(name: str, extents: Tuple[int, ...], memory: Layout, threads: int, vector: int) -> TvLayout:
    runs = memory.flat_modes()
    weights = _colex_weights([e for e, _ in runs])
    by_address = sorted(range(len(runs)), key=lambda i: (runs[i][1], i))
    contiguous = 1
    for i in by_address:
        extent, stride = runs[i]
        if extent == 1:
            continue
        if stride != contiguous:
            break
        contiguous *= extent
    if vector > contiguous or contiguous % vector:
        raise LayoutIncompatible(f"vector of {vector} elements does not divide the contiguous run of "
                                 f"{contiguous} in {name}")
    total = math.prod(extents)
    if total % (vector * threads):
        raise NonDivisibleTile(f"{name}: {total} elements not divisible by {threads} threads x {vector}-element "
                               f"vectors")
    reps = total // (vector * threads)
    # address rank -> logical index, then (thread, (vector lane, repeat)) -> address rank
    rank_to_logical = Layout(tuple(runs[i][0] for i in by_address), tuple(weights[i] for i in by_address))
    rank_of_tv = Layout(((threads,), (vector, reps)), ((vector,), (1, vector * threads)))
    return TvLayout(compose(rank_to_logical, rank_of_tv), extents)


def coalesced_access_layout(decl: TensorDecl, memory_layout: Optional[Layout], threads: int,
                            vector_elems: int) -> TvLayout:
    """Copy anchor: walk memory in address order (dimensions by ascending stride); each thread
    takes ``vector_elems`` contiguous elements, consecutive threads consecutive vectors, repeats
    after all threads. The vector must divide the stride-1 contiguous run."""
    extents = tuple(decl.shape)
    memory = memory_layout if memory_layout is not None else Layout(extents, _colex_weights(extents))
    return _coalesced(decl.name, extents, memory, threads, vector_elems)


def _warp_grid(op: OpNode, warps: int, rm: int, rn: int) -> Tuple[int, int, Layout]:
    """(warps along rows, along columns, grid coordinate -> warp id)."""
    arrangement = op.thread_arrangement
    if arrangement is None:
        wm = math.gcd(warps, rm)
        wn = warps // wm
        grid = Layout((wm, wn), (1, wm))
    else:
        if arrangement.rank != 2:
            raise ShapeMismatch("thread arrangement must have two modes")
        wm, wn = (math.prod(e for e, _ in _runs(arrangement, i)) for i in (0, 1))
        if wm * wn != warps:
            raise NonDivisibleTile(f"thread arrangement uses {wm * wn} warps, have {warps}")
        grid = arrangement
    if rm % wm or rn % wn:
        raise NonDivisibleTile(f"warp grid {wm}x{wn} does not divide the {rm}x{rn} tile grid")
    return wm, wn, grid


@functools.lru_cache(maxsize=1024)
def _gemm_anchor(mnk: Tuple[int, int, int], inst: Instruction, warps: int, arrangement: Optional[Layout]):
    M, N, K = mnk
    MI, NI, KI = inst.mnk
    if M % MI or N % NI or K % KI:
        raise NonDivisibleTile(f"gemm {M}x{N}x{K} not divisible by instruction tile {MI}x{NI}x{KI}")
    rm, rn, kreps = M // MI, N // NI, K // KI
    probe = OpNode("gemm", [], [], thread_arrangement=arrangement)
    wm, wn, grid = _warp_grid(probe, warps, rm, rn)
    warp_order = inverse(grid)            # warp id -> grid position (rows fastest)

    def placed(tv: TvLayout, rows: int) -> Layout:
        """Instruction fragment re-addressed into a tile with ``rows`` rows."""
        return compose(Layout(tv.tile, (1, rows)), tv.layout)

    def warp_runs(row_step: int, col_step: int):
        return compose(Layout((wm, wn), (row_step, col_step)), warp_order).flat_modes()

    frag_a, frag_b, frag_c = inst.mma_layouts()
    fa, fb, fc = placed(frag_a, M), placed(frag_b, N), placed(frag_c, M)
    row_rep, col_rep = (rm // wm, MI * wm), (rn // wn, M * NI * wn)
    c_tv = tv_from_mode_lists(_runs(fc, 0) + warp_runs(MI, M * NI), _runs(fc, 1) + [row_rep, col_rep], (M, N))
    a_tv = tv_from_mode_lists(_runs(fa, 0) + warp_runs(MI, 0), _runs(fa, 1) + [row_rep, (kreps, M * KI)], (M, K))
    b_tv = tv_from_mode_lists(_runs(fb, 0) + warp_runs(0, NI), _runs(fb, 1) + [(rn // wn, NI * wn), (kreps, N * KI)],
                              (N, K))
    return a_tv, b_tv, c_tv


def init_gemm_anchor(op: OpNode, graph: ProgramGraph, inst: Instruction, config: SynthesisConfig
                     ) -> Dict[str, TvLayout]:
    """Tile C with the instruction's fragments (warps over rows first unless annotated; per-thread
    repeats in the value mode: rows, then columns / reduction) and derive A and B from it."""
    a, b, _ = (graph.tensor(n) for n in op.operands)
    (M, K), N = a.shape, b.shape[0]
    tvs = _gemm_anchor((M, N, K), inst, config.warps, op.thread_arrangement)
    return dict(zip(op.operands, tvs))


# ------------------------------------------------------------------------------------------ solving
@functools.lru_cache(maxsize=1 << 14)
def _solve_copy(known: TvLayout, inst: Instruction, dtype: DType, known_is_src: bool) -> TvLayout:
    src_inst, dst_inst = inst.copy_layouts(dtype)
    mine, theirs = (src_inst, dst_inst) if known_is_src else (dst_inst, src_inst)
    ti, vi = mine.threads, mine.values
    if known.threads < ti or known.threads % ti:
        raise LayoutIncompatible(f"{inst.name} needs {ti} threads; layout has {known.threads}")
    if known.values < vi or known.values % vi:
        raise LayoutIncompatible(f"{inst.name} moves {vi} values/thread; layout has {known.values}")
    try:
        inner_known, outer_t, outer_v = restrict_tv(known, ti, vi)
        tile_to_tv = compose(inner_known.layout, inverse(mine.layout))
        other = compose(tile_to_tv, theirs.layout)
    except (NotDivisible, NotInvertible, OutOfDomain) as e:
        raise LayoutIncompatible(str(e)) from e
    return tv_from_mode_lists(_runs(other, 0) + outer_t, _runs(other, 1) + outer_v, known.tile)


def solve_copy(known: TvLayout, inst: Instruction, dtype, known_is_src: bool) -> TvLayout:
    """The other side of a copy: ``g = f o p^-1 o q`` on one instruction tile (the known side
    restricted to the instruction's threads x values); outer thread / value digits carry over."""
    return _solve_copy(known, inst, dtype, known_is_src)


def reduce_projection(extents: Tuple[int, ...], dim: int) -> Layout:
    """Input linear index -> output linear index with dimension ``dim`` collapsed."""
    out = tuple(1 if i == dim else e for i, e in enumerate(extents))
    weights = _colex_weights(out)
    return Layout(tuple(extents), tuple(0 if i == dim else w for i, w in enumerate(weights)))


def solve_reduce(f: TvLayout, dim: int) -> TvLayout:
    out = tuple(1 if i == dim else e for i, e in enumerate(f.tile))
    return TvLayout(compose(reduce_projection(f.tile, dim), f.layout), out)


# ------------------------------------------------------------------------------------- constraints
_GEMM_PAIRS = (("gemm_rows", (2, 0)), ("gemm_cols", (2, 1)), ("gemm_red", (0, 1)))


def build_constraints(component: Sequence[OpNode], graph: ProgramGraph) -> List[TvConstraint]:
    """Three per matrix op (rows C~A, columns C~B, reduction A~B), one per copy (R->R: element
    equality), cast / elementwise (element equality) and reduce."""
    out: List[TvConstraint] = []
    for op in component:
        if op.kind == "gemm":
            for kind, (i, j) in _GEMM_PAIRS:
                pair = [op.operands[i], op.operands[j]]
                out.append(TvConstraint(kind, op, list(pair), list(pair)))
            continue
        if op.kind == "copy":
            names = [op.operands[0], op.results[0]]
            both_reg = all(graph.tensor(n).scope == "Register" for n in names)
            kind = "elem" if both_reg else "copy"
        elif op.kind in ("cast", "elementwise"):
            names, kind = op.operands + op.results, "elem"
        elif op.kind == "reduce":
            names, kind = [op.operands[0], op.results[0]], "reduce"
        else:
            continue
        out.append(TvConstraint(kind, op, [slot_for(graph, op, n) for n in names], names))
    return out


class PropagationState:
    """Slot -> layout (first assignment wins) and the redistribution patches conflicts produced."""

    def __init__(self, graph: ProgramGraph, config: SynthesisConfig):
        self.graph = graph
        self.config = config
        self.layouts: Dict[SlotKey, TvLayout] = {}
        self.patches: List[RearrangePatch] = []
        self._views: Dict[Tuple[int, str], TvLayout] = {}

    def effective(self, slot: SlotKey, tensor: str, op: OpNode) -> TvLayout:
        """The layout ``op`` sees for ``tensor`` (its patch, if it has one)."""
        return self._views.get((op.index, tensor)) or self.layouts[slot]

    def assign(self, slot: SlotKey, tensor: str, layout: TvLayout, op: OpNode) -> None:
        held = self.layouts.setdefault(slot, layout)
        if held is layout or held.same_function(layout):
            return
        self.patches.append(RearrangePatch(op.index, tensor, held, layout))
        self._views[(op.index, tensor)] = layout


def _anchor_copy(component: Sequence[OpNode], graph: ProgramGraph) -> Tuple[OpNode, str, Optional[Layout]]:
    """The copy moving the most bytes, global-backed copies first, then op order."""
    def rank(op: OpNode):
        src, dst = graph.tensor(op.operands[0]), graph.tensor(op.results[0])
        side = op.operands[0] if src.scope == "Global" else op.results[0] if dst.scope == "Global" else None
        return (0 if side else 1, -src.bytes, op.index), side

    ranked = sorted((rank(op) + (op,) for op in component if op.kind == "copy"), key=lambda r: r[0])
    if not ranked:
        raise UnsolvedResidual("component has no copy to anchor")
    _, side, op = ranked[0]
    if side is None:
        return op, op.operands[0], None
    return op, side, graph.tensor(side).layout


def _seed(component, graph, choices, config, catalog, state) -> None:
    gemms = [op for op in component if op.kind == "gemm"]
    for op in gemms:
        a, b, c = (graph.tensor(n) for n in op.operands)
        inst = choices.get(op.index) or fastest_mma(catalog, a.dtype, b.dtype, c.dtype)
        choices[op.index] = inst
        for name, tv in init_gemm_anchor(op, graph, inst, config).items():
            state.assign(name, name, tv, op)
    if not gemms:
        op, tensor, memory = _anchor_copy(component, graph)
        decl = graph.tensor(tensor)
        inst = choices.get(op.index)
        tv = coalesced_access_layout(decl, memory, config.threads, inst.vector_elems(decl.dtype) if inst else 1)
        state.assign(slot_for(graph, op, tensor), tensor, tv, op)
    for op in component:   # user-written rearrange targets are fixed too
        if op.kind == "rearrange" and op.rearrange_target is not None:
            out = op.results[0]
            state.assign(out, out, TvLayout(op.rearrange_target, graph.tensor(out).shape), op)


def _discharge(c: TvConstraint, graph: ProgramGraph, choices: Dict[int, Instruction], state: PropagationState):
    if c.kind.startswith("gemm"):
        return  # satisfied by construction of the anchor
    first = next((i for i, s in enumerate(c.slots) if s in state.layouts), None)
    if first is None:
        raise UnsolvedResidual(f"op {c.op.index}: no known layout to solve from")
    known = state.effective(c.slots[first], c.tensors[first], c.op)
    if c.kind == "elem":
        for slot, name in zip(c.slots, c.tensors):
            state.assign(slot, name, TvLayout(known.layout, graph.tensor(name).shape), c.op)
    elif c.kind == "copy":
        inst = choices.get(c.op.index)
        if inst is None:
            raise NoInstructionAvailable(f"op {c.op.index}: no instruction chosen for copy")
        solved = solve_copy(known, inst, graph.tensor(c.tensors[first]).dtype, first == 0)
        other = 1 - first
        state.assign(c.slots[other], c.tensors[other], TvLayout(solved.layout, graph.tensor(c.tensors[other]).shape),
                     c.op)
    elif c.kind == "reduce":
        if c.slots[0] not in state.layouts:
            raise UnsolvedResidual(f"op {c.op.index}: reduction input has no layout; reductions solve forward only")
        source = state.effective(c.slots[0], c.tensors[0], c.op)
        state.assign(c.slots[1], c.tensors[1], solve_reduce(source, c.op.reduce_dim), c.op)
    else:
        raise UnsolvedResidual(f"unknown constraint kind {c.kind}")


def propagate(component: Sequence[OpNode], graph: ProgramGraph, choices: Dict[int, Instruction],
              config: SynthesisConfig, catalog: Catalog, state: PropagationState,
              constraint_order: Optional[Sequence[int]] = None) -> None:
    """Seed the anchors, then solve in rounds until nothing is left (or nothing is ready)."""
    todo = build_constraints(component, graph)
    if constraint_order is not None:
        todo = [todo[i] for i in constraint_order]
    _seed(component, graph, choices, config, catalog, state)
    while todo:
        ready = [c for c in todo if sum(s not in state.layouts for s in c.slots) <= 1]
        if not ready:
            break
        for c in ready:
            _discharge(c, graph, choices, state)
            c.solved = True
        todo = [c for c in todo if not c.solved]
    if todo:
        raise UnsolvedResidual("constraints left unsolved (no anchor reaches them): "
                               + ", ".join(f"op {c.op.index} ({c.op.kind})" for c in todo))
