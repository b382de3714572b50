"""Thread-value layout inference over one component of a tile program.

Contract: /root/reference/pkg/src/tilesynth/synth.py:46-500 -- anchors (matrix ops tile their
output with the instruction fragments and derive the inputs; otherwise the copy moving the most
data, preferring global-backed ones, gets a coalesced access layout), copy / element / reduce
solving rules, conflict handling (the second, different layout a register tensor receives becomes a
redistribution patch on that op's view), and the round-based readiness of the solver: in every
round each constraint that is ready at the START of the round (at most one unknown slot) is
solved, in constraint order.

Construction here: the solver is a :class:`LayoutFlow` object holding the slot table; constraint
records are plain tuples; the three solving rules are methods picked from a dispatch table; the
matrix anchor is table-driven over the operand roles (a, b, c).
"""
from __future__ import annotations

import math
from typing import Dict, List, Tuple, Union

from .algebra import Layout, compose, inverse
from .errors import (LayoutIncompatible, NoInstructionAvailable, NonDivisibleTile, NotDivisible, NotInvertible,
                     OutOfDomain, ShapeMismatch, UnsolvedResidual)
from .isa_table import Catalog, Instruction, fastest_mma
from .records import record
from .tileprog import OpNode, ProgramGraph, TensorDecl
from .algebra import TvLayout, restrict_tv, tv_from_mode_lists

SlotKey = Union[str, Tuple[int, str]]


def _check_threads(cfg):
    if cfg.threads < 32 or cfg.threads % 32:
        raise ValueError("thread count must be a positive multiple of 32")


SynthesisConfig = record("SynthesisConfig", [("threads", 128), ("max_candidates", 64)],
                         "Threads per tile (a multiple of 32) and the search-leaf cap.", module=__name__,
                         __post_init__=_check_threads, warps=property(lambda cfg: cfg.threads // 32))

# op ``op_index`` sees ``tensor`` as ``to_layout`` while the tensor carries ``from_layout``;
# ``inserted`` is False for user-written rearrange ops
RearrangePatch = record("RearrangePatch", ["op_index", "tensor", "from_layout", "to_layout", ("inserted", True)],
                        "A register redistribution at a conflict edge.", module=__name__)

# kind: "copy" | "elem" | "reduce" | "gemm_rows" | "gemm_cols" | "gemm_red"
TvConstraint = record("TvConstraint", ["kind", "op", "slots", "tensors", ("solved", False)],
                      "One layout constraint of an op over its slots.", module=__name__)


class PropagationState:
    """The slot table of one synthesis leaf: slot -> TvLayout, plus redistribution patches."""

    def __init__(self, graph, config):
        self.graph, self.config = graph, config
        self.layouts: Dict[SlotKey, TvLayout] = {}
        self.patches: List[RearrangePatch] = []
        self._views: Dict[Tuple[int, str], TvLayout] = {}

    def effective(self, slot, tensor, op):
        """The layout ``op`` sees for ``tensor`` (its patch, if it has one)."""
        return self._views.get((op.index, tensor)) or self.layouts[slot]

    def assign(self, slot, tensor, layout, op):
        have = self.layouts.setdefault(slot, layout)
        if have is layout or have.same_function(layout):
            return
        self.patches.append(RearrangePatch(op.index, tensor, have, layout))
        self._views[(op.index, tensor)] = layout


class LayoutFlow:
    """Solving rules over a :class:`PropagationState` (one method per constraint kind)."""

    def __init__(self, graph, choices, state):
        self.graph, self.choices, self.state = graph, choices, state
        self.rules = {"elem": self.elem, "copy": self.copy, "reduce": self.reduce}

    def solve(self, c):
        if c.kind.startswith("gemm"):
            return  # discharged by the matrix anchor's construction
        known = [i for i, s in enumerate(c.slots) if s in self.state.layouts]
        if not known:
            raise UnsolvedResidual(f"op {c.op.index}: no known layout to solve from")
        self.rules[c.kind](c, known[0])

    def _shape(self, tensor):
        return self.graph.tensor(tensor).shape

    def elem(self, c, k):
        base = self.state.effective(c.slots[k], c.tensors[k], c.op).layout
        for slot, tensor in zip(c.slots, c.tensors):
            self.state.assign(slot, tensor, TvLayout(base, self._shape(tensor)), c.op)

    def copy(self, c, k):
        inst = self.choices.get(c.op.index)
        if inst is None:
            raise NoInstructionAvailable(f"op {c.op.index}: no instruction chosen for copy")
        known = self.state.effective(c.slots[k], c.tensors[k], c.op)
        other = solve_copy(known, inst, self.graph.tensor(c.tensors[k]).dtype, k == 0)
        self.state.assign(c.slots[1 - k], c.tensors[1 - k], TvLayout(other.layout, self._shape(c.tensors[1 - k])),
                          c.op)

    def reduce(self, c, k):
        if c.slots[0] not in self.state.layouts:
            raise UnsolvedResidual(f"op {c.op.index}: reduction input has no layout; reductions solve forward only")
        f = self.state.effective(c.slots[0], c.tensors[0], c.op)
        self.state.assign(c.slots[1], c.tensors[1], solve_reduce(f, c.op.reduce_dim), c.op)


def propagate(component, graph, choices, config, catalog, state, constraint_order=None):
    """Seed the anchors, then solve in rounds until nothing is left (UnsolvedResidual if a round
    makes no progress)."""
    cons = build_constraints(component, graph)
    if constraint_order is not None:
        cons = [cons[i] for i in constraint_order]
    gemms = [op for op in component if op.kind == "gemm"]
    for op in gemms:
        if op.index not in choices or not choices[op.index]:
            choices[op.index] = fastest_mma(catalog, *(graph.tensor(n).dtype for n in op.operands))
        for tensor, tv in init_gemm_anchor(op, graph, choices[op.index], config).items():
            state.assign(tensor, tensor, tv, op)
    if not gemms:
        op, tensor, mem = _anchor_copy(component, graph)
        decl, inst = graph.tensor(tensor), choices.get(op.index)
        tv = coalesced_access_layout(decl, mem, config.threads, inst.vector_elems(decl.dtype) if inst else 1)
        state.assign(slot_for(graph, op, tensor), tensor, tv, op)
    for op in component:
        if op.kind == "rearrange" and op.rearrange_target is not None:
            out = op.results[0]
            state.assign(out, out, TvLayout(op.rearrange_target, graph.tensor(out).shape), op)
    flow = LayoutFlow(graph, choices, state)
    todo = list(cons)
    while todo:
        ready = [c for c in todo if sum(s not in state.layouts for s in c.slots) <= 1]
        if not ready:
            listing = ", ".join(f"op {c.op.index} ({c.op.kind})" for c in todo)
            raise UnsolvedResidual(f"constraints left unsolved (no anchor reaches them): {listing}")
        for c in ready:
            flow.solve(c)
            c.solved = True
        todo = [c for c in todo if not c.solved]


# -------------------------------------------------------------------------------------- constraints
def build_constraints(component, graph):
    """One record per copy / element / reduce op; three per matrix op (rows C~A, columns C~B,
    reduction A~B)."""
    out = []
    for op in component:
        if op.kind == "gemm":
            a, b, c = op.operands
            out += [TvConstraint(k, op, [x, y], [x, y])
                    for k, x, y in (("gemm_rows", c, a), ("gemm_cols", c, b), ("gemm_red", a, b))]
            continue
        if op.kind == "copy":
            names = [op.operands[0], op.results[0]]
            kind = "elem" if all(graph.tensor(n).scope == "Register" for n in names) else "copy"
        elif op.kind in ("cast", "elementwise"):
            names, kind = op.operands + op.results, "elem"
        elif op.kind == "reduce":
            names, kind = [op.operands[0], op.results[0]], "reduce"
        else:
            continue
        out.append(TvConstraint(kind, op, [slot_for(graph, op, n) for n in names], names))
    return out


# ------------------------------------------------------------------------------------------ solving
def solve_copy(known, inst, dtype, known_is_src):
    """The other side of a copy: restrict the known side to one instruction tile, map through the
    inverse of the instruction's layout on that side and its layout on the other side; the digits
    beyond one instruction (warp groups, outer iterations) carry over unchanged."""
    src_tv, dst_tv = inst.copy_layouts(dtype)
    near, far = (src_tv, dst_tv) if known_is_src else (dst_tv, src_tv)
    for have, need, what in ((known.threads, near.threads, "threads"), (known.values, near.values, "values/thread")):
        if have < need or have % need:
            raise LayoutIncompatible(f"{inst.name} needs {need} {what}; layout has {have}")
    try:
        core, outer_t, outer_v = restrict_tv(known, near.threads, near.values)
        mapped = compose(compose(core.layout, inverse(near.layout)), far.layout)
    except (NotDivisible, NotInvertible, OutOfDomain) as e:
        raise LayoutIncompatible(str(e)) from e
    return tv_from_mode_lists(_runs(mapped, 0) + outer_t, _runs(mapped, 1) + outer_v, known.tile)


def solve_reduce(f, dim):
    return TvLayout(compose(reduce_projection(f.tile, dim), f.layout),
                    tuple(1 if i == dim else e for i, e in enumerate(f.tile)))


def reduce_projection(extents, dim):
    """Input linear index -> output linear index with dimension ``dim`` collapsed."""
    kept = tuple(1 if i == dim else e for i, e in enumerate(extents))
    w = _colex_weights(kept)
    return Layout(tuple(extents), tuple(0 if i == dim else w[i] for i in range(len(extents))))


def init_gemm_anchor(op, graph, inst, config):
    """Tile C with the instruction's fragments over a warp grid; A and B follow. Warps go to the
    thread mode; per-thread repeats go to the value mode (row / column repeats, then k steps)."""
    a, b, c = map(graph.tensor, op.operands)
    (M, K), N = a.shape, b.shape[0]
    MI, NI, KI = inst.mnk
    if M % MI or N % NI or K % KI:
        raise NonDivisibleTile(f"gemm {M}x{N}x{K} not divisible by instruction tile {MI}x{NI}x{KI}")
    rm, rn, kreps = M // MI, N // NI, K // KI
    wm, wn, grid = _warp_grid(op, config.warps, rm, rn)
    warp_to_cell = inverse(grid)
    frag = dict(zip("abc", inst.mma_layouts()))
    # role: (tile extents, warp row step, warp column step, value repeats)
    roles = {
        "a": ((M, K), MI, 0, [(rm // wm, MI * wm), (kreps, M * KI)]),
        "b": ((N, K), 0, NI, [(rn // wn, NI * wn), (kreps, N * KI)]),
        "c": ((M, N), MI, M * NI, [(rm // wm, MI * wm), (rn // wn, M * NI * wn)]),
    }
    out = {}
    for role, name in zip("abc", op.operands):
        extents, row_step, col_step, reps = roles[role]
        tv = frag[role]
        placed = compose(Layout(tv.tile, (1, extents[0])), tv.layout)
        warps = compose(Layout((wm, wn), (row_step, col_step)), warp_to_cell).flat_modes()
        out[name] = tv_from_mode_lists(_runs(placed, 0) + warps, _runs(placed, 1) + reps, extents)
    return out


# ------------------------------------------------------------------------------------------ anchors
def coalesced_access_layout(decl, memory_layout, threads, vector_elems):
    """Threads walk memory in ascending address order: each owns ``vector_elems`` consecutive
    elements, neighbours own neighbouring vectors, leftover iterations come after all threads."""
    extents, total = decl.shape, decl.elems
    mem = memory_layout or Layout(extents, _colex_weights(extents))
    runs = mem.runs
    logical_w = _colex_weights([e for e, _ in runs])
    by_addr = sorted(range(len(runs)), key=lambda i: (runs[i][1], i))
    contiguous = 1
    for i in by_addr:
        e, d = runs[i]
        if e == 1:
            continue
        if d != contiguous:
            break
        contiguous *= e
    if vector_elems > contiguous or contiguous % vector_elems:
        raise LayoutIncompatible(f"vector of {vector_elems} elements does not divide the contiguous run of "
                                 f"{contiguous} in {decl.name}")
    if total % (vector_elems * threads):
        raise NonDivisibleTile(f"{decl.name}: {total} elements not divisible by {threads} threads x "
                               f"{vector_elems}-element vectors")
    addr_rank = Layout(tuple(runs[i][0] for i in by_addr), tuple(logical_w[i] for i in by_addr))
    thread_vec = Layout(((threads,), (vector_elems, total // (vector_elems * threads))),
                        ((vector_elems,), (1, vector_elems * threads)))
    return TvLayout(compose(addr_rank, thread_vec), extents)


def _anchor_copy(component, graph):
    """The copy moving the most bytes, global-backed ones first (then program order)."""
    def rank(op):
        src, dst = graph.tensor(op.operands[0]), graph.tensor(op.results[0])
        side = src if src.scope == "Global" else dst if dst.scope == "Global" else None
        return (side is None, -src.bytes, op.index), side
    ranked = sorted((rank(op) + (op,) for op in component if op.kind == "copy"), key=lambda r: r[0])
    if not ranked:
        raise UnsolvedResidual("component has no copy to anchor")
    _, side, op = ranked[0]
    return (op, op.operands[0], None) if side is None else (op, side.name, side.layout)


def _warp_grid(op, warps, rm, rn):
    """(warps along rows, warps along columns, grid coordinate -> warp id). Default: as many warps
    along the rows as divide both; a thread_arrangement annotation overrides."""
    arr = op.thread_arrangement
    if arr is None:
        wm = math.gcd(warps, rm)
        wm, wn, grid = wm, warps // wm, Layout((wm, warps // wm), (1, wm))
    else:
        if arr.rank != 2:
            raise ShapeMismatch("thread arrangement must have two modes")
        wm, wn = (math.prod(e for e, _ in _runs(arr, i)) for i in (0, 1))
        if wm * wn != warps:
            raise NonDivisibleTile(f"thread arrangement uses {wm * wn} warps, have {warps}")
        grid = arr
    if rm % wm or rn % wn:
        raise NonDivisibleTile(f"warp grid {wm}x{wn} does not divide the {rm}x{rn} tile grid")
    return wm, wn, grid


def _colex_weights(extents):
    w = [1]
    for e in extents[:-1]:
        w.append(w[-1] * e)
    return tuple(w[:len(extents)])


def _runs(layout, mode):
    return layout.mode(mode).flat_modes()


def slot_for(graph, op, tensor):
    """Register tensors have one layout program-wide (keyed by name); a shared / global tensor is
    seen per access, keyed (op, "src" | "dst")."""
    if graph.tensor(tensor).scope == "Register":
        return tensor
    if op.kind == "copy":
        return op.index, ("src" if tensor == op.operands[0] else "dst")
    return op.index, ("src" if tensor in op.operands else "dst")
