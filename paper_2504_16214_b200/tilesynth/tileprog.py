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
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Tuple

from . import ituple
from .algebra import Layout, parse_layout
from .errors import ArityError, ParseError, TileSynthError, UnknownTensor


# ------------------------------------------------------------------------------------------- dtypes
@dataclass(frozen=True)
class DType:
    kind: str                         # "float" | "int" | "uint"
    bits: int
    float_format: Optional[str] = None

    @property
    def name(self):
        return f"float8_{self.float_format}" if self.float_format else f"{self.kind}{self.bits}"

    def __str__(self):
        return self.name


_DTYPES: Dict[str, DType] = dict(
    [(f"float{b}", DType("float", b)) for b in (16, 32, 64)]
    + [("bfloat16", DType("float", 16))]
    + [(f"{k}{b}", DType(k, b)) for b in (1, 2, 4, 8, 16, 32, 64) for k in ("int", "uint")]
    + [(f"float8_{f}", DType("float", 8, f)) for f in ("e5m2", "e4m3")])


def parse_dtype(name):
    if name not in _DTYPES:
        raise ParseError(f"unknown dtype {name!r}")
    return _DTYPES[name]


# ------------------------------------------------------------------------------------------ tensors
SCOPES = ("Global", "Shared", "Register")
ACTION_KINDS = ("copy", "gemm", "cast", "rearrange", "elementwise", "reduce")
_DERIVING = ("cast", "rearrange", "elementwise", "reduce")   # ops that declare their result


@dataclass
class TensorDecl:
    name: str
    scope: str
    dtype: DType
    shape: Tuple[int, ...]
    layout: Optional[Layout] = None   # Global tensors only
    buffer: Optional[str] = None      # backing buffer of a Global tensor

    @property
    def elems(self):
        return math.prod(self.shape)

    @property
    def bytes(self):
        return self.elems * self.dtype.bits / 8


@dataclass
class OpNode:
    kind: str
    operands: List[str]               # tensors read
    results: List[str]                # tensors written
    index: int = -1
    line: int = 0
    trip_count: int = 1               # product of the enclosing loop trip counts
    cast_dtype: Optional[DType] = None
    reduce_dim: Optional[int] = None
    rearrange_target: Optional[Layout] = None
    elementwise_fn: Optional[str] = None
    thread_arrangement: Optional[Layout] = None

    @property
    def tensors(self):
        return self.operands + [r for r in self.results if r not in self.operands]


@dataclass
class ProgramGraph:
    tensors: Dict[str, TensorDecl]
    ops: List[OpNode]
    diagnostics: List[str] = field(default_factory=list)

    def tensor(self, name):
        if name not in self.tensors:
            raise UnknownTensor(f"unknown tensor {name!r}")
        return self.tensors[name]

    def producers(self, name):
        return [op for op in self.ops if name in op.results]

    def consumers(self, name):
        return [op for op in self.ops if name in op.operands]


# ------------------------------------------------------------------------------------------ parsing
class _Reader:
    """Parser state: declarations, ops, the open loops and pending annotations."""

    def __init__(self):
        self.tensors: Dict[str, TensorDecl] = {}
        self.ops: List[OpNode] = []
        self.loops: List[int] = []
        self.notes: List[Tuple[int, int, Layout]] = []
        self.line = 0

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


_STATEMENTS: Dict[str, Tuple[bool, Optional[Tuple[int, ...]], str, Callable]] = {
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


def copy_src_dst(graph, op):
    if op.kind != "copy":
        raise ArityError(f"op {op.index} is not a copy")
    return graph.tensor(op.operands[0]), graph.tensor(op.results[0])


# --------------------------------------------------------------------------------------- validation
def _tensor_rules(name, t):
    out = []
    if t.dtype.bits < 8 and t.shape[0] * t.dtype.bits < 8:
        out.append(f"tensor {name}: sub-byte dtype {t.dtype} needs an innermost run of >= "
                   f"{8 // t.dtype.bits} elements, got {t.shape[0]}")
    if t.scope == "Global":
        if t.layout is None:
            out.append(f"tensor {name}: Global tensors require a layout")
        elif any(d == 0 for e, d in t.layout.runs if e > 1):
            out.append(f"tensor {name}: broadcast (stride-0) global layouts unsupported")
    return out


def _need_register(g, op, name, role):
    return [] if g.tensor(name).scope == "Register" else [f"op {op.index}: {role} must be Register"]


def _check_copy(g, op):
    src, dst = copy_src_dst(g, op)
    out = []
    if src.shape != dst.shape:
        out.append(f"op {op.index}: copy shape mismatch {src.name}{src.shape} -> {dst.name}{dst.shape}")
    if src.dtype.bits != dst.dtype.bits:
        out.append(f"op {op.index}: copy dtype width mismatch {src.dtype} -> {dst.dtype}")
    return out


def _check_gemm(g, op):
    a, b, c = map(g.tensor, op.operands)
    out = []
    for t in (a, b, c):
        out += _need_register(g, op, t.name, f"gemm operand {t.name}")
        if len(t.shape) != 2:
            out.append(f"op {op.index}: gemm operand {t.name} must be rank-2")
    if all(len(t.shape) == 2 for t in (a, b, c)):
        (m, ka), (n, kb) = a.shape, b.shape
        if ka != kb:
            out.append(f"op {op.index}: gemm reduction extent mismatch between {a.name} (K={ka}) and "
                       f"{b.name} (K={kb})")
        if c.shape != (m, n):
            out.append(f"op {op.index}: gemm output extent mismatch {c.name}{c.shape} vs ({m},{n})")
    return out


def _check_reduce(g, op):
    src = g.tensor(op.operands[0])
    out = []
    if op.reduce_dim is None or not 0 <= op.reduce_dim < len(src.shape):
        out.append(f"op {op.index}: reduce dim {op.reduce_dim} out of range for rank-{len(src.shape)} "
                   f"tensor {src.name}")
    return out + _need_register(g, op, src.name, "reduce operand")


def _check_elementwise(g, op):
    shapes = {g.tensor(n).shape for n in op.operands}
    return [f"op {op.index}: elementwise operand shapes differ: {shapes}"] if len(shapes) > 1 else []


def _check_rearrange(g, op):
    out = _need_register(g, op, op.operands[0], "rearrange operand")
    if op.rearrange_target is not None and op.rearrange_target.rank != 2:
        out.append(f"op {op.index}: rearrange target must be a two-mode (thread, value) layout")
    return out


_OP_RULES = {
    "copy": _check_copy,
    "gemm": _check_gemm,
    "cast": lambda g, op: _need_register(g, op, op.operands[0], "cast operand"),
    "reduce": _check_reduce,
    "elementwise": _check_elementwise,
    "rearrange": _check_rearrange,
}


def validate(graph):
    """Scope / type / shape rules; returns the diagnostics (empty = valid)."""
    diags = [d for name, t in graph.tensors.items() for d in _tensor_rules(name, t)]
    written = set()
    for op in graph.ops:
        if op.kind in _DERIVING:
            diags += [f"op {op.index}: tensor {r} produced twice" for r in op.results if r in written]
        diags += _OP_RULES.get(op.kind, lambda g, o: [])(graph, op)
        written.update(op.results)
    written = set()
    produced_somewhere = {r for op in graph.ops for r in op.results}
    for op in graph.ops:
        for name in op.operands:
            if (graph.tensor(name).scope == "Register" and name in produced_somewhere
                    and name not in written and name not in op.results):
                diags.append(f"op {op.index}: tensor {name} used before definition")
        written.update(op.results)
    return diags


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


__all__ = ["DType", "TensorDecl", "OpNode", "ProgramGraph", "parse_dtype", "parse_program", "print_program",
           "validate", "eliminate_dead_code", "partition_components", "copy_src_dst", "SCOPES", "ACTION_KINDS",
           "TileSynthError"]
