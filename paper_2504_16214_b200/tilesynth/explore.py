"""Candidate search over the copy-instruction choices, per-candidate shared / staging buffer
synthesis, and the one-call pipeline (validate -> dead code -> search -> rank).

Contract: /root/reference/pkg/src/tilesynth/synth.py:66-75,505-720 and pipeline.py:1-60 -- leaves in
depth-first (lexicographic) order of the per-copy choice indices, capped at ``max_candidates - 1``
walked leaves plus the all-narrowest fallback leaf; leaves failing layout solving or buffer
unification are pruned; failures surface as diagnostics.

Construction here: a leaf is evaluated component by component, and each component's propagation
result is memoised on the instruction choices of ITS copies (components only share shared-memory
buffers, which are synthesised afterwards), so a search of n leaves over c components propagates
each distinct (component, choice) pair once. The leaf walk is ``itertools.product`` over the
choice lists.

Candidates are ranked by the analytical latency model at the end of the module (contract
/root/reference/pkg/src/tilesynth/cost.py:1-274: the step sequence with redistributions and
rearranges inlined as staging store/load pairs, per-thread invocation counts, read-after-write
stalls, ranking by total cycles then discovery order). A step waits for the results it reads,
occupies the issue path for (invocations x issue cycles x bank-conflict replays) and completes
``completion_cycles`` after its issue ends; the timing pass is a scoreboard -- a map from tensor to
the latest completion time of its in-flight writers.
"""
from __future__ import annotations

import itertools
from collections import namedtuple
from typing import Dict, List, Optional, Sequence, Tuple

from .algebra import TvLayout
from .errors import (LayoutIncompatible, NoInstructionAvailable, NonDivisibleTile, NotDivisible, NotInvertible,
                     OutOfDomain, ShapeMismatch, StrideConflict, TileSynthError, Unsatisfiable)
from .isa_table import Catalog, Instruction, candidates_for_copy
from .layout_flow import PropagationState, RearrangePatch, SlotKey, SynthesisConfig, propagate
from .records import record
from .smem_plan import BufferCopy, SmemLayout, synthesize_buffer
from .tileprog import OpNode, ProgramGraph, TensorDecl, eliminate_dead_code, partition_components, validate

PRUNE = (LayoutIncompatible, NonDivisibleTile, NotDivisible, NotInvertible, OutOfDomain, ShapeMismatch,
         StrideConflict, Unsatisfiable, NoInstructionAvailable)


# ``cost`` is filled in by :func:`estimate`
Candidate = record("Candidate", ["index", "choices", "layouts", "patches", "smem", ("staging", dict), ("cost", None)],
                   "One surviving search leaf: instruction per op, layout per slot, patches, buffers.",
                   module=__name__)


class _ComponentMemo:
    """Propagation results of one component, keyed by the instruction choices of its ops."""

    def __init__(self, ops):
        self.ops = list(ops)
        self.indices = [op.index for op in ops]
        self.seen: Dict[Tuple, object] = {}

    def run(self, graph, choices, config, catalog):
        key = tuple(id(choices.get(i)) for i in self.indices)
        hit = self.seen.get(key)
        if hit is None:
            state = PropagationState(graph, config)
            local = {i: choices[i] for i in self.indices if i in choices}
            try:
                propagate(self.ops, graph, local, config, catalog, state)
                hit = (local, state.layouts, state.patches)
            except TileSynthError as e:
                hit = e
            self.seen[key] = hit
        if isinstance(hit, Exception):
            raise hit
        return hit


class _Evaluator:
    """Evaluates leaves of one search (graph, catalog, config fixed)."""

    def __init__(self, graph, catalog, config):
        self.graph, self.catalog, self.config = graph, catalog, config
        self.parts = [_ComponentMemo(c) for c in partition_components(graph)]

    def evaluate(self, picked):
        choices = dict(picked)
        state = PropagationState(self.graph, self.config)
        for part in self.parts:
            chosen, layouts, patches = part.run(self.graph, choices, self.config, self.catalog)
            choices.update(chosen)
            state.layouts.update(layouts)
            state.patches.extend(patches)
        return (choices, state.layouts, state.patches, _synthesize_shared(self.graph, choices, state),
                _synthesize_staging(self.graph, self.catalog, self.config, state))


# ------------------------------------------------------------------------------------------ pipeline
SynthesisResult = record(
    "SynthesisResult", ["graph", "config", "catalog", ("diagnostics", list), ("candidates", list)],
    "The live graph, the ranked candidates (best first) or the diagnostics.", module=__name__,
    ok=property(lambda r: not r.diagnostics and (bool(r.candidates) or not r.graph.ops)),
    best=property(lambda r: r.candidates[0] if r.candidates else None))


# ----------------------------------------------------------------------------------------
# latency model and ranking
class CostOp(namedtuple("CostOp", "label reads writes instruction invocations issue_cycles completion_cycles "
                                "replays", defaults=(1,))):
    """One issue step: the tensors it reads and writes (RAW tracking) and its latency. ``replays``:
    an n-way bank-conflicted access occupies the issue path n times."""

    __slots__ = ()

    @property
    def issue_total(self):
        return self.invocations * self.issue_cycles * self.replays


# one row of the timing pass: the step, its issue cycles, stall, start and completion time
OpCost = namedtuple("OpCost", "label instruction invocations issue stall start completes")


class CostEstimate:
    """Total modelled cycles of a candidate and the per-step timing rows."""

    def __init__(self, total_cycles, breakdown=None):
        self.total_cycles, self.breakdown = total_cycles, list(breakdown or [])

    def render(self):
        fmt = "{0.label}: issue {0.issue} (x{0.invocations}), stall {0.stall}, start {0.start}, completes {0.completes}"
        return [fmt.format(c) for c in self.breakdown] + ["total %d" % self.total_cycles]


def _step_rearrange(op, cand, graph, catalog, alu):
    out_tv = cand.layouts.get(op.results[0])
    staged = _staging_ops("rearrange@%d" % op.index, op.operands[0], out_tv.values if out_tv else 1, catalog, cand,
                          op.trip_count)
    return staged + [_op_step(op, "rearrange", "register_move", 1)]


def _step_copy(op, cand, graph, catalog, alu):
    inst = cand.choices.get(op.index)
    if inst is None:  # register -> register move, one ALU op per value
        return [_op_step(op, "copy", alu, cand.layouts[op.results[0]].values * op.trip_count)]
    buffers = [cand.smem[t] for t in (op.operands[0], op.results[0]) if t in cand.smem]
    replays = max([1] + [b.copy_conflicts.get(op.index, 1) for b in buffers])
    return [_op_step(op, "copy", inst, count_invocations(op, cand, inst, graph), replays)]


def _step_gemm(op, cand, graph, catalog, alu):
    inst = cand.choices[op.index]
    return [_op_step(op, "gemm", inst, count_invocations(op, cand, inst, graph))]


_STEPS = {"rearrange": _step_rearrange, "copy": _step_copy, "gemm": _step_gemm}


def synthesize_program(graph, catalog, config=None):
    """Validate, drop dead code, search, rank. Failures come back as diagnostics (``result.ok``)."""
    config = config or SynthesisConfig()
    problems = validate(graph)
    if problems:
        return SynthesisResult(graph, config, catalog, problems)
    live = eliminate_dead_code(graph)
    if graph.ops and not live.ops:
        return SynthesisResult(live, config, catalog, ["all operations are dead code (no global store)"])
    try:
        found = expand_search(live, catalog, config)
    except TileSynthError as e:
        return SynthesisResult(live, config, catalog, [str(e)])
    if live.ops and not found:
        return SynthesisResult(live, config, catalog, ["no valid candidate: every instruction assignment failed"])
    return SynthesisResult(live, config, catalog, [], rank(found, live, catalog))


def expand_search(graph, catalog, config):
    """Surviving leaves in lexicographic order of the choice indices (at most ``max_candidates - 1``
    from the walk, at least one), then the all-narrowest fallback leaf if it was not among them."""
    if not graph.ops:
        return []
    points = _copy_choice_points(graph, catalog)
    ev = _Evaluator(graph, catalog, config)
    found = []
    kept = set()

    def leaf(pick):
        try:
            parts = ev.evaluate({op.index: opts[i] for (op, opts), i in zip(points, pick)})
        except PRUNE:
            return None
        return Candidate(len(found), *parts)

    cap = max(1, config.max_candidates - 1)
    for pick in itertools.product(*(range(len(opts)) for _, opts in points)):
        if len(found) >= cap:
            break
        cand = leaf(pick)
        if cand is not None:
            found.append(cand)
            kept.add(pick)
    narrowest = tuple(len(opts) - 1 for _, opts in points)
    if config.max_candidates > 1 and narrowest not in kept:
        cand = leaf(narrowest)
        if cand is not None:
            found.append(cand)
    return found


def evaluate_assignment(graph, catalog, config, choices):
    """Propagate layouts over every component and synthesise every buffer for one leaf;
    ``choices`` is completed in place with the matrix instructions the anchors pick."""
    state = PropagationState(graph, config)
    for component in partition_components(graph):
        propagate(component, graph, choices, config, catalog, state)
    return (choices, state.layouts, state.patches, _synthesize_shared(graph, choices, state),
            _synthesize_staging(graph, catalog, config, state))


def rank(candidates, graph, catalog):
    """Ascending total cycles; ties keep discovery order."""
    for cand in candidates:
        if cand.cost is None:
            estimate(cand, graph, catalog)
    return sorted(candidates, key=lambda c: (c.cost.total_cycles, c.index))


def estimate(candidate, graph, catalog):
    candidate.cost = estimate_sequence(cost_sequence(candidate, graph, catalog))
    return candidate.cost


# ------------------------------------------------------------------------------------------ timing
def estimate_sequence(seq):
    """Issue the steps in order against a scoreboard of tensor -> latest pending completion."""
    ready, clock, horizon, rows = {}, 0, 0, []
    for step in seq:
        begin = max([clock] + [ready[t] for t in step.reads if t in ready])
        stall, clock = begin - clock, begin + step.issue_total
        finish = clock + step.completion_cycles
        ready.update((t, max(ready.get(t, 0), finish)) for t in step.writes)
        horizon = max(horizon, finish)
        rows.append(OpCost(step.label, step.instruction, step.invocations, step.issue_total, stall, begin, finish))
    return CostEstimate(max(clock, horizon), rows)


def cost_sequence(candidate, graph, catalog):
    """The candidate's steps in program order; an op's redistribution patches run just before it."""
    alu = catalog.alu()
    seq = []
    for op in graph.ops:
        for p in candidate.patches:
            if p.op_index == op.index:
                seq += _staging_ops(f"redistribute@{p.op_index}:{p.tensor}", p.tensor, p.to_layout.values, catalog,
                                    candidate, op.trip_count)
        seq += _STEPS.get(op.kind, _step_alu)(op, candidate, graph, catalog, alu)
    return seq


# ------------------------------------------------------------------------------------- invocations
def count_invocations(op, candidate, inst, graph):
    """Per-thread instruction invocations of one op, loop trip counts included."""
    lay = candidate.layouts
    if op.kind == "copy":
        tv = (lay.get((op.index, "src")) or lay.get(op.operands[0]) or lay.get((op.index, "dst"))
              or lay[op.results[0]])
        vec = inst.vector_elems(graph.tensor(op.operands[0]).dtype)
        if tv.values % vec:
            raise NonDivisibleTile(f"op {op.index}: {tv.values} values/thread not divisible by {vec}-element vectors")
        return tv.values // vec * op.trip_count
    if op.kind == "gemm":
        (m, k), n = graph.tensor(op.operands[0]).shape, graph.tensor(op.operands[1]).shape[0]
        mi, ni, ki = inst.mnk
        per_issue = mi * ni * ki * (lay[op.operands[2]].threads // 32)
        if (m * n * k) % per_issue:
            raise NonDivisibleTile(f"op {op.index}: ragged matrix tiling")
        return m * n * k // per_issue * op.trip_count
    return lay[op.results[0]].values * op.trip_count   # register-file op: one per produced value


def _step_alu(op, cand, graph, catalog, alu):
    return [_op_step(op, op.kind, alu, count_invocations(op, cand, alu, graph))]


def _op_step(op, what, inst, count, replays=1):
    """The step of op ``op`` itself (label ``op<i>.<what>``), reading its operands, writing its results."""
    name, issue, done = (inst, 1, 1) if isinstance(inst, str) else (inst.name, inst.issue_cycles,
                                                                    inst.completion_cycles)
    return CostOp("op%d.%s" % (op.index, what), set(op.operands), set(op.results), name, count, issue, done, replays)


# --------------------------------------------------------------------------------------- sequences
def _staging_ops(label, tensor, values, catalog, candidate, trip):
    """A redistribution = store to + load from a staging buffer (scalar 16-bit round trip when no
    staging layout was synthesised)."""
    buf = f"<{label}>"
    staging = candidate.staging.get(label)
    if staging is not None and len(staging.copies) == 2:
        legs = [(bc.instruction, max(1, values // bc.vector_elems), staging.copy_conflicts.get(bc.op_index, 1))
                for bc in staging.copies]
    else:
        legs = [("sts_16", values, 1), ("lds_16", values, 1)]
    flow = (({tensor}, {buf}, "store"), ({buf}, {tensor}, "load"))
    out = []
    for (name, inv, replays), (reads, writes, leg) in zip(legs, flow):
        inst = catalog.by_name.get(name)
        out.append(CostOp(f"{label}.{leg}", reads, writes, name, inv * trip, inst.issue_cycles if inst else 2,
                          inst.completion_cycles if inst else 22, replays))
    return out


def _synthesize_staging(graph, catalog, config, state):
    """A staging buffer for every user rearrange and every inserted redistribution patch: the first
    (store, load) pair whose two accesses unify."""
    jobs = [(f"rearrange@{op.index}", op.operands[0], state.layouts[op.operands[0]], state.layouts[op.results[0]])
            for op in graph.ops
            if op.kind == "rearrange" and op.operands[0] in state.layouts and op.results[0] in state.layouts]
    jobs += [(f"redistribute@{p.op_index}:{p.tensor}", p.tensor, p.from_layout, p.to_layout) for p in state.patches]
    out = {}
    for label, tensor, before, after in jobs:
        decl = graph.tensor(tensor)
        for st, ld in _staging_instructions(catalog, decl):
            pair = [BufferCopy(-1, before, st.vector_elems(decl.dtype), st.name),
                    BufferCopy(-2, after, ld.vector_elems(decl.dtype), ld.name)]
            try:
                out[label] = synthesize_buffer(label, decl.shape, decl.dtype.bits, pair)
                break
            except PRUNE:
                continue
        else:
            raise Unsatisfiable(f"no staging layout for redistribution of {tensor}")
    return out


def _staging_instructions(catalog, decl):
    """(store, load) pairs of equal width for a register redistribution through shared memory,
    widest store first; loads are generic entries."""
    tmp = TensorDecl("staging", "Shared", decl.dtype, decl.shape)
    loads = {}
    for ld in candidates_for_copy(catalog, tmp, decl):
        if ld.generic:
            loads.setdefault(ld.vector_bytes, ld)
    return [(st, loads[st.vector_bytes]) for st in candidates_for_copy(catalog, decl, tmp) if st.vector_bytes in loads]


def _synthesize_shared(graph, choices, state):
    """One layout + swizzle per shared tensor from the accesses of every copy touching it."""
    users = {}
    for op in graph.ops:
        if op.kind != "copy":
            continue
        for side, name in (("src", op.operands[0]), ("dst", op.results[0])):
            decl = graph.tensor(name)
            if decl.scope == "Shared":
                inst = choices[op.index]
                users.setdefault(name, []).append(BufferCopy(op.index, state.layouts[(op.index, side)],
                                                             inst.vector_elems(decl.dtype), inst.name))
    return {name: synthesize_buffer(name, graph.tensor(name).shape, graph.tensor(name).dtype.bits, copies)
            for name, copies in sorted(users.items())}


def _copy_choice_points(graph, catalog):
    """(copy op, its candidate instructions) for every copy that needs an instruction."""
    out = []
    for op in graph.ops:
        if op.kind == "copy":
            src, dst = graph.tensor(op.operands[0]), graph.tensor(op.results[0])
            if not src.scope == dst.scope == "Register":
                out.append((op, candidates_for_copy(catalog, src, dst)))
    return out
