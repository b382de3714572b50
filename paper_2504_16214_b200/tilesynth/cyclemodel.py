"""Analytical latency model: a candidate is a sequence of issue steps; a step waits for the results
it reads, occupies the issue path for (invocations x issue cycles x bank-conflict replays), and
completes ``completion_cycles`` after its issue ends; the total adds the last completion.

Contract: /root/reference/pkg/src/tilesynth/cost.py:1-274 (the step sequence with redistributions
and rearranges inlined as staging store/load pairs, per-thread invocation counts, read-after-write
stalls, ranking by total cycles then discovery order). Construction here: the step list is built
by a per-kind table of step makers, and the timing pass is a scoreboard -- a map from tensor to the
latest completion time of its in-flight writers -- instead of a list of in-flight records.
"""
from __future__ import annotations

from collections import namedtuple

from .errors import NonDivisibleTile


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


def _op_step(op, what, inst, count, replays=1):
    """The step of op ``op`` itself (label ``op<i>.<what>``), reading its operands, writing its results."""
    name, issue, done = (inst, 1, 1) if isinstance(inst, str) else (inst.name, inst.issue_cycles,
                                                                    inst.completion_cycles)
    return CostOp("op%d.%s" % (op.index, what), set(op.operands), set(op.results), name, count, issue, done, replays)


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


def _step_alu(op, cand, graph, catalog, alu):
    return [_op_step(op, op.kind, alu, count_invocations(op, cand, alu, graph))]


_STEPS = {"rearrange": _step_rearrange, "copy": _step_copy, "gemm": _step_gemm}


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


def estimate(candidate, graph, catalog):
    candidate.cost = estimate_sequence(cost_sequence(candidate, graph, catalog))
    return candidate.cost


def rank(candidates, graph, catalog):
    """Ascending total cycles; ties keep discovery order."""
    for cand in candidates:
        if cand.cost is None:
            estimate(cand, graph, catalog)
    return sorted(candidates, key=lambda c: (c.cost.total_cycles, c.index))
