"""Tile programs: the text format, the program graph, validation, dead-code elimination and the
split into register-connected components.

Contract: /root/reference/pkg/src/tilesynth/ir.py:1-552 -- the statement syntax, the op numbering
(action statements only, program order), loop trip counts, annotations, the validator's
diagnostics (their text is part of the synthesis report), dead-code and partition semantics.

Construction here: statements are parsed by a table of small handlers keyed on the statement
word (each declares its own arity / lhs rule); validation is a set of per-tensor rules and a
per-kind dispatch table; liveness is a backward worklist from the global stores; components are a
breadth-first walk over the op <-> register-tensor incidence graph.

    t = global_view <buffer> <dtype> <layout>      t = register_tensor <dtype> <shape>
    t = shared_tensor <dtype> <shape>              copy <src> <dst>
    gemm <c> <a> <b>                               t2 = cast <t1> <dtype>
    t2 = rearrange <t1> [<tv-layout>]              t = elementwise <fn> <t1> ... <tn>
    t2 = reduce <t1> <dim>                         loop <n> ... endloop
    annotate <op-index> thread_arrangement <layout>
"""
from __future__ import annotations

import math
from collections import deque

from . import ituple
from .algebra import Layout, parse_layout
from .errors import ArityError, ParseError, TileSynthError, UnknownTensor
from .records import record


# ----------------------------------------------------------------------------------- record types
DType = record(
    "DType", ["kind", "bits", ("float_format", None)],
    "An element type: kind 'float' | 'int' | 'uint', width in bits, fp8 flavour.", frozen=True, module=__name__,
    name=property(lambda d: f"float8_{d.float_format}" if d.float_format else f"{d.kind}{d.bits}"),
    __str__=lambda d: d.name)

_DTYPES = {}
for _b in (16, 32, 64):
    _DTYPES[f"float{_b}"] = DType("float", _b)
_DTYPES["bfloat16"] = DType("float", 16)
for _b in (1, 2, 4, 8, 16, 32, 64):
    _DTYPES.update({f"{_k}{_b}": DType(_k, _b) for _k in ("int", "uint")})
_DTYPES.update({f"float8_{_f}": DType("float", 8, _f) for _f in ("e5m2", "e4m3")})


SCOPES = ("Global", "Shared", "Register")
ACTION_KINDS = ("copy", "gemm", "cast", "rearrange", "elementwise", "reduce")
_DERIVING = ("cast", "rearrange", "elementwise", "reduce")   # ops that declare their result

# a Global tensor also carries its layout and backing buffer name
TensorDecl = record(
    "TensorDecl", ["name", "scope", "dtype", "shape", ("layout", None), ("buffer", None)],
    "A declared tensor: scope, element type, logical extents (+ layout / buffer when Global).", module=__name__,
    elems=property(lambda t: math.prod(t.shape)),
    bytes=property(lambda t: math.prod(t.shape) * t.dtype.bits / 8))

# one action statement; trip_count = product of the enclosing loop trip counts; the per-kind extras
# (cast dtype, reduce dim, rearrange target, elementwise fn) and the annotation default to None
OpNode = record(
    "OpNode", ["kind", "operands", "results", ("index", -1), ("line", 0), ("trip_count", 1), ("cast_dtype", None),
               ("reduce_dim", None), ("rearrange_target", None), ("elementwise_fn", None),
               ("thread_arrangement", None)],
    "An action statement: the tensors it reads (operands) and writes (results).", module=__name__,
    tensors=property(lambda op: op.operands + [r for r in op.results if r not in op.operands]))


def _tensor_of(graph, name):
    if name not in graph.tensors:
        raise UnknownTensor(f"unknown tensor {name!r}")
    return graph.tensors[name]


ProgramGraph = record(
    "ProgramGraph", ["tensors", "ops", ("diagnostics", list)],
    "Declarations by name, action statements in program order, diagnostics.", module=__name__,
    tensor=_tensor_of,
    producers=lambda g, name: [op for op in g.ops if name in op.results],
    consumers=lambda g, name: [op for op in g.ops if name in op.operands])


# ------------------------------------------------------------------------------------------ parsing
class _Reader:
    """Parser state: declarations, ops, the open loops and pending annotations."""

    def __init__(self):
        self.tensors, self.ops, self.loops, self.notes, self.line = {}, [], [], [], 0

    def fail(self, msg):
        raise ParseError(msg, self.line)

    def known(self, name):
        if name not in self.tensors:
            self.fail(f"unknown tensor {name!r}")
        return self.tensors[name]

    def declare(self, name, scope, dtype, shape, **extra):
        if name in self.tensors:
            self.fail(f"tensor {name!r} redeclared")
        self.tensors[name] = TensorDecl(name, scope, dtype, tuple(shape), **extra)

    def emit(self, kind, reads, writes, **extra):
        self.ops.append(OpNode(kind, reads, writes, line=self.line, trip_count=math.prod(self.loops), **extra))

    def layout(self, text):
        try:
            return parse_layout(text)
        except ParseError as e:
            self.fail(str(e))

    def integer(self, text, what):
        try:
            return int(text)
        except ValueError:
            self.fail(f"{what} must be an integer: {text}")

    def shape(self, text):
        try:
            tree = ituple.parse_tuple(text)
        except ParseError as e:
            self.fail(str(e))
        if min(ituple.leaves(tree)) < 1:
            self.fail(f"shape extents must be >= 1: {text}")
        return (tree,) if isinstance(tree, int) else tuple(map(ituple.size, tree))


# handler(reader, lhs, args); the tuple before it: (needs lhs?, allowed arg counts or None = any>=2, usage)
def _global_view(r, lhs, args):
    lay = r.layout(args[2])
    r.declare(lhs, "Global", parse_dtype(args[1]), map(ituple.size, lay.shape), layout=lay, buffer=args[0])


def _local_tensor(scope):
    def handler(r, lhs, args):
        r.declare(lhs, scope, parse_dtype(args[0]), r.shape(args[1]))
    return handler


def _copy(r, lhs, args):
    r.emit("copy", [r.known(args[0]).name], [r.known(args[1]).name])


def _gemm(r, lhs, args):
    c, a, b = (r.known(x).name for x in args)
    r.emit("gemm", [a, b, c], [c])


def _cast(r, lhs, args):
    src = r.known(args[0])
    dtype = parse_dtype(args[1])
    r.declare(lhs, src.scope, dtype, src.shape)
    r.emit("cast", [src.name], [lhs], cast_dtype=dtype)


def _rearrange(r, lhs, args):
    src = r.known(args[0])
    target = r.layout(args[1]) if len(args) > 1 else None
    r.declare(lhs, src.scope, src.dtype, src.shape)
    r.emit("rearrange", [src.name], [lhs], rearrange_target=target)


def _elementwise(r, lhs, args):
    ins = [r.known(a).name for a in args[1:]]
    first = r.tensors[ins[0]]
    r.declare(lhs, first.scope, first.dtype, first.shape)
    r.emit("elementwise", ins, [lhs], elementwise_fn=args[0])


def _reduce(r, lhs, args):
    src = r.known(args[0])
    dim = r.integer(args[1], "reduce dim")
    shape = [1 if i == dim else s for i, s in enumerate(src.shape)]
    r.declare(lhs, src.scope, src.dtype, shape)
    r.emit("reduce", [src.name], [lhs], reduce_dim=dim)


def _loop(r, lhs, args):
    n = r.integer(args[0], "loop trip count")
    if n < 1:
        r.fail("loop trip count must be >= 1")
    r.loops.append(n)


def _endloop(r, lhs, args):
    if not r.loops:
        r.fail("endloop without matching loop")
    r.loops.pop()


def _annotate(r, lhs, args):
    if args[1] != "thread_arrangement":
        r.fail("usage: annotate <op-index> thread_arrangement <layout>")
    r.notes.append((r.line, r.integer(args[0], "op index"), r.layout(args[2])))


_STATEMENTS = {  # word -> (needs lhs?, allowed arg counts (None = any >= 2), usage, handler)
    "global_view": (True, (3,), "t = global_view <buffer> <dtype> <layout>", _global_view),
    "register_tensor": (True, (2,), "t = register_tensor <dtype> <shape>", _local_tensor("Register")),
    "shared_tensor": (True, (2,), "t = shared_tensor <dtype> <shape>", _local_tensor("Shared")),
    "copy": (False, (2,), "copy <src> <dst>", _copy),
    "gemm": (False, (3,), "gemm <c> <a> <b>", _gemm),
    "cast": (True, (2,), "t2 = cast <t1> <dtype>", _cast),
    "rearrange": (True, (1, 2), "t2 = rearrange <t1> [<tv-layout>]", _rearrange),
    "elementwise": (True, None, "t = elementwise <fn> <t1> ... <tn>", _elementwise),
    "reduce": (True, (2,), "t2 = reduce <t1> <dim>", _reduce),
    "loop": (False, (1,), "loop <trip-count>", _loop),
    "endloop": (False, (0,), "endloop", _endloop),
    "annotate": (False, (3,), "annotate <op-index> thread_arrangement <layout>", _annotate),
}


# --------------------------------------------------------------------------------------- validation
# The diagnostics are part of the synthesis report, so their wording is the reference's
# (ir.py:379-480); the checks below only pick a message and its fields.
_MESSAGES = {
    "subbyte": "tensor {t}: sub-byte dtype {dt} needs an innermost run of >= {need} elements, got {run}",
    "no_layout": "tensor {t}: Global tensors require a layout",
    "broadcast": "tensor {t}: broadcast (stride-0) global layouts unsupported",
    "twice": "op {i}: tensor {t} produced twice",
    "copy_shape": "op {i}: copy shape mismatch {s}{ss} -> {d}{ds}",
    "copy_width": "op {i}: copy dtype width mismatch {sd} -> {dd}",
    "not_register": "op {i}: {role} must be Register",
    "rank2": "op {i}: gemm operand {t} must be rank-2",
    "gemm_k": "op {i}: gemm reduction extent mismatch between {a} (K={ka}) and {b} (K={kb})",
    "gemm_out": "op {i}: gemm output extent mismatch {c}{cs} vs ({m},{n})",
    "reduce_dim": "op {i}: reduce dim {dim} out of range for rank-{r} tensor {t}",
    "elem_shapes": "op {i}: elementwise operand shapes differ: {shapes}",
    "rearrange_rank": "op {i}: rearrange target must be a two-mode (thread, value) layout",
    "before_def": "op {i}: tensor {t} used before definition",
}


def _reg(g, op, name, role):
    if g.tensor(name).scope != "Register":
        yield "not_register", dict(i=op.index, role=role)


def _copy_findings(g, op):
    src, dst = copy_src_dst(g, op)
    if src.shape != dst.shape:
        yield "copy_shape", dict(i=op.index, s=src.name, ss=src.shape, d=dst.name, ds=dst.shape)
    if src.dtype.bits != dst.dtype.bits:
        yield "copy_width", dict(i=op.index, sd=src.dtype, dd=dst.dtype)


def _gemm_findings(g, op):
    ts = [g.tensor(n) for n in op.operands]
    for t in ts:
        yield from _reg(g, op, t.name, f"gemm operand {t.name}")
        if len(t.shape) != 2:
            yield "rank2", dict(i=op.index, t=t.name)
    if {len(t.shape) for t in ts} == {2}:
        a, b, c = ts
        if a.shape[1] != b.shape[1]:
            yield "gemm_k", dict(i=op.index, a=a.name, ka=a.shape[1], b=b.name, kb=b.shape[1])
        if c.shape != (a.shape[0], b.shape[0]):
            yield "gemm_out", dict(i=op.index, c=c.name, cs=c.shape, m=a.shape[0], n=b.shape[0])


def _reduce_findings(g, op):
    src = g.tensor(op.operands[0])
    if op.reduce_dim is None or not 0 <= op.reduce_dim < len(src.shape):
        yield "reduce_dim", dict(i=op.index, dim=op.reduce_dim, r=len(src.shape), t=src.name)
    yield from _reg(g, op, src.name, "reduce operand")


def _elementwise_findings(g, op):
    shapes = {g.tensor(n).shape for n in op.operands}
    if len(shapes) > 1:
        yield "elem_shapes", dict(i=op.index, shapes=shapes)


def _rearrange_findings(g, op):
    yield from _reg(g, op, op.operands[0], "rearrange operand")
    if op.rearrange_target is not None and op.rearrange_target.rank != 2:
        yield "rearrange_rank", dict(i=op.index)


_OP_FINDINGS = {
    "copy": _copy_findings,
    "gemm": _gemm_findings,
    "cast": lambda g, op: _reg(g, op, op.operands[0], "cast operand"),
    "reduce": _reduce_findings,
    "elementwise": _elementwise_findings,
    "rearrange": _rearrange_findings,
}


__all__ = ["DType", "TensorDecl", "OpNode", "ProgramGraph", "parse_dtype", "parse_program", "print_program",
           "validate", "eliminate_dead_code", "partition_components", "copy_src_dst", "SCOPES", "ACTION_KINDS",
           "TileSynthError"]


def parse_program(text):
    """Program text -> graph with resolved declarations (ParseError carries the line)."""
    r = _Reader()
    lines = text.splitlines()
    for r.line, raw in enumerate(lines, start=1):
        stmt = raw.split("#", 1)[0].strip()
        if not stmt:
            continue
        lhs, _, rhs = stmt.partition("=") if "=" in stmt else (None, "", stmt)
        lhs = lhs.strip() if lhs is not None else None
        words = rhs.split()
        if not words:
            r.fail("empty statement")
        spec = _STATEMENTS.get(words[0])
        if spec is None:
            r.fail(f"unknown statement {words[0]!r}")
        wants_lhs, counts, usage, handler = spec
        args = words[1:]
        arity_ok = len(args) >= 2 if counts is None else len(args) in counts
        if (lhs is not None) != wants_lhs or not arity_ok:
            r.fail(f"usage: {usage}")
        handler(r, lhs, args)
    if r.loops:
        raise ParseError("unterminated loop", len(lines))
    for i, op in enumerate(r.ops):
        op.index = i
    for line, idx, lay in r.notes:
        if not 0 <= idx < len(r.ops):
            raise ParseError(f"annotate index {idx} out of range", line)
        r.ops[idx].thread_arrangement = lay
    return ProgramGraph(r.tensors, r.ops)


def print_program(graph):
    """Canonical text: declarations, then one statement per op (looped ops wrapped in their own
    ``loop n`` / ``endloop``), then the annotations; parse(print(g)) prints identically."""
    made = {r for op in graph.ops if op.kind in _DERIVING for r in op.results}
    decl_fmt = {
        "Global": lambda t: f"{t.name} = global_view {t.buffer} {t.dtype} {t.layout}",
        "Shared": lambda t: f"{t.name} = shared_tensor {t.dtype} {ituple.format_tuple(t.shape)}",
        "Register": lambda t: f"{t.name} = register_tensor {t.dtype} {ituple.format_tuple(t.shape)}",
    }
    out = [decl_fmt[t.scope](t) for t in graph.tensors.values() if t.scope in decl_fmt and t.name not in made]
    op_fmt = {
        "copy": lambda op: f"copy {op.operands[0]} {op.results[0]}",
        "gemm": lambda op: "gemm {2} {0} {1}".format(*op.operands),
        "cast": lambda op: f"{op.results[0]} = cast {op.operands[0]} {op.cast_dtype}",
        "rearrange": lambda op: f"{op.results[0]} = rearrange {op.operands[0]}"
                                + (f" {op.rearrange_target}" if op.rearrange_target else ""),
        "elementwise": lambda op: f"{op.results[0]} = elementwise {op.elementwise_fn} {' '.join(op.operands)}",
        "reduce": lambda op: f"{op.results[0]} = reduce {op.operands[0]} {op.reduce_dim}",
    }
    for op in graph.ops:
        if op.kind in op_fmt:
            body = op_fmt[op.kind](op)
            out.append(body if op.trip_count == 1 else f"loop {op.trip_count}\n{body}\nendloop")
    out += [f"annotate {op.index} thread_arrangement {op.thread_arrangement}"
            for op in graph.ops if op.thread_arrangement is not None]
    return "\n".join(out) + "\n"


def validate(graph):
    """Scope / type / shape rules; returns the diagnostics (empty = valid)."""
    return [_MESSAGES[key].format(**fields) for key, fields in _findings(graph)]


# -------------------------------------------------------------------------------------- dead code
def eliminate_dead_code(graph):
    """Keep the ops from which a copy into a Global tensor is reachable (backward liveness over the
    tensors they write); renumber the survivors; keep live and Global declarations."""
    live_ops = {op.index for op in graph.ops
                if op.kind == "copy" and graph.tensor(op.results[0]).scope == "Global"}
    live = {t for op in graph.ops if op.index in live_ops for t in op.tensors}
    writers = {}
    for op in graph.ops:
        for r in op.results:
            writers.setdefault(r, []).append(op)
    todo = deque(live)
    while todo:
        for op in writers.get(todo.popleft(), ()):
            if op.index not in live_ops:
                live_ops.add(op.index)
                fresh = [t for t in op.tensors if t not in live]
                live.update(fresh)
                todo.extend(fresh)
    kept = [op for op in graph.ops if op.index in live_ops]
    for i, op in enumerate(kept):
        op.index = i
    return ProgramGraph({n: d for n, d in graph.tensors.items() if n in live or d.scope == "Global"}, kept,
                        list(graph.diagnostics))


# -------------------------------------------------------------------------------------- components
def partition_components(graph):
    """Ops connected through register tensors (shared tensors cut the graph), in first-op order,
    program order inside a component."""
    touching = {}
    for op in graph.ops:
        for name in op.tensors:
            if graph.tensor(name).scope == "Register":
                touching.setdefault(name, []).append(op.index)
    by_op = {}
    for name, idxs in touching.items():
        for i in idxs:
            by_op.setdefault(i, []).append(name)
    owner = {}
    for op in graph.ops:
        if op.index in owner:
            continue
        owner[op.index] = op.index
        todo = deque([op.index])
        while todo:
            for name in by_op.get(todo.popleft(), ()):
                for j in touching[name]:
                    if j not in owner:
                        owner[j] = op.index
                        todo.append(j)
    groups = {}
    for op in graph.ops:
        groups.setdefault(owner[op.index], []).append(op)
    return list(groups.values())


def copy_src_dst(graph, op):
    if op.kind != "copy":
        raise ArityError(f"op {op.index} is not a copy")
    return graph.tensor(op.operands[0]), graph.tensor(op.results[0])


def parse_dtype(name):
    if name not in _DTYPES:
        raise ParseError(f"unknown dtype {name!r}")
    return _DTYPES[name]


def _findings(graph):
    for name, t in graph.tensors.items():
        yield from _tensor_findings(name, t)
    written = set()
    for op in graph.ops:
        if op.kind in _DERIVING:
            for r in op.results:
                if r in written:
                    yield "twice", dict(i=op.index, t=r)
        yield from _OP_FINDINGS.get(op.kind, lambda g, o: ())(graph, op)
        written.update(op.results)
    produced_somewhere = {r for op in graph.ops for r in op.results}
    written = set()
    for op in graph.ops:
        for name in op.operands:
            if (graph.tensor(name).scope == "Register" and name in produced_somewhere
                    and name not in written and name not in op.results):
                yield "before_def", dict(i=op.index, t=name)
        written.update(op.results)


def _tensor_findings(name, t):
    if t.dtype.bits < 8 and t.shape[0] * t.dtype.bits < 8:
        yield "subbyte", dict(t=name, dt=t.dtype, need=8 // t.dtype.bits, run=t.shape[0])
    if t.scope == "Global" and t.layout is None:
        yield "no_layout", dict(t=name)
    elif t.scope == "Global" and any(d == 0 for e, d in t.layout.runs if e > 1):
        yield "broadcast", dict(t=name)
