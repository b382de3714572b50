"""Tile-program IR: dtypes, tensor declarations, operations, the text format, and the graph passes
(validation, dead-code elimination, register-connected components).

Text format and pass semantics are the reference's (``/root/reference/pkg/src/tilesynth/ir.py``:
statements ``:1-20``, ``parse_program`` ``:163-315``, ``validate`` ``:379-480``,
``eliminate_dead_code`` ``:486-514``, ``partition_components`` ``:520-552``); the diagnostics text is
part of the report contract and is kept verbatim. Structure here: statement handlers are a
dispatch table over a small parser state object; validation is a list of rule functions;
liveness is a backward worklist; components are a breadth-first walk of the op/tensor graph.
"""
from __future__ import annotations

from collections import deque
from dataclasses import dataclass, field
from typing import Callable, Dict, Iterator, List, Optional, Tuple

from . import nested
from .errors import ArityError, ParseError, UnknownTensor
from .layout_algebra import Layout, parse_layout


# ------------------------------------------------------------------------------------------ dtypes
@dataclass(frozen=True)
class DType:
    kind: str            # "float" | "int" | "uint"
    bits: int
    float_format: Optional[str] = None

    @property
    def name(self) -> str:
        return f"float8_{self.float_format}" if self.float_format else f"{self.kind}{self.bits}"

    def __str__(self) -> str:
        return self.name


def _dtype_table() -> Dict[str, DType]:
    table = {f"float{b}": DType("float", b) for b in (16, 32, 64)}
    table["bfloat16"] = DType("float", 16)  # an alias: equal to, and printed as, float16
    for b in (1, 2, 4, 8, 16, 32, 64):
        table[f"int{b}"], table[f"uint{b}"] = DType("int", b), DType("uint", b)
    table.update({f"float8_{f}": DType("float", 8, f) for f in ("e5m2", "e4m3")})
    return table


_DTYPES = _dtype_table()


def parse_dtype(name: str) -> DType:
    if name not in _DTYPES:
        raise ParseError(f"unknown dtype {name!r}")
    return _DTYPES[name]


SCOPES = ("Global", "Shared", "Register")
ACTION_KINDS = ("copy", "gemm", "cast", "rearrange", "elementwise", "reduce")
_DERIVED = ("cast", "rearrange", "elementwise", "reduce")   # ops that declare their result


@dataclass
class TensorDecl:
    name: str
    scope: str
    dtype: DType
    shape: Tuple[int, ...]
    layout: Optional[Layout] = None   # Global tensors only
    buffer: Optional[str] = None      # Global tensors: backing buffer name

    @property
    def elems(self) -> int:
        return nested.size(tuple(self.shape))

    @property
    def bytes(self) -> float:
        return self.elems * self.dtype.bits / 8


@dataclass
class OpNode:
    kind: str
    operands: List[str]
    results: List[str]
    index: int = -1
    line: int = 0
    trip_count: int = 1
    cast_dtype: Optional[DType] = None
    reduce_dim: Optional[int] = None
    rearrange_target: Optional[Layout] = None
    elementwise_fn: Optional[str] = None
    thread_arrangement: Optional[Layout] = None

    @property
    def tensors(self) -> List[str]:
        return self.operands + [r for r in self.results if r not in self.operands]


@dataclass
class ProgramGraph:
    tensors: Dict[str, TensorDecl]
    ops: List[OpNode]
    diagnostics: List[str] = field(default_factory=list)

    def tensor(self, name: str) -> TensorDecl:
        decl = self.tensors.get(name)
        if decl is None:
            raise UnknownTensor(f"unknown tensor {name!r}")
        return decl

    def producers(self, name: str) -> List[OpNode]:
        return [op for op in self.ops if name in op.results]

    def consumers(self, name: str) -> List[OpNode]:
        return [op for op in self.ops if name in op.operands]


# ------------------------------------------------------------------------------------------ parser
class _Parse:
    """Mutable state of one parse: the tensor table, the op list, open loops, annotations."""

    def __init__(self):
        self.tensors: Dict[str, TensorDecl] = {}
        self.ops: List[OpNode] = []
        self.loops: List[int] = []
        self.notes: List[Tuple[int, int, Layout]] = []
        self.line = 0

    def fail(self, message: str):
        raise ParseError(message, self.line)

    def trip(self) -> int:
        n = 1
        for count in self.loops:
            n *= count
        return n

    def name(self, tensor: str) -> str:
        if tensor not in self.tensors:
            self.fail(f"unknown tensor {tensor!r}")
        return tensor

    def decl(self, tensor: str) -> TensorDecl:
        return self.tensors[self.name(tensor)]

    def declare(self, decl: TensorDecl) -> None:
        if decl.name in self.tensors:
            self.fail(f"tensor {decl.name!r} redeclared")
        self.tensors[decl.name] = decl

    def emit(self, kind: str, operands, results, **extra) -> None:
        self.ops.append(OpNode(kind, list(operands), list(results), line=self.line, trip_count=self.trip(), **extra))

    def layout(self, text: str) -> Layout:
        try:
            return parse_layout(text)
        except ParseError as e:
            raise ParseError(str(e), self.line) from None

    def int_arg(self, text: str, what: str) -> int:
        try:
            return int(text)
        except ValueError:
            raise ParseError(f"{what}: {text}", self.line) from None

    def shape(self, text: str) -> Tuple[int, ...]:
        try:
            tree = nested.parse_tuple(text)
        except ParseError as e:
            raise ParseError(str(e), self.line) from None
        if any(x < 1 for x in nested.leaves(tree)):
            self.fail(f"shape extents must be >= 1: {text}")
        return (tree,) if isinstance(tree, int) else tuple(nested.size(m) for m in tree)


def _st_global_view(p: _Parse, lhs, args):
    layout = p.layout(args[2])
    p.declare(TensorDecl(lhs, "Global", parse_dtype(args[1]), tuple(nested.size(m) for m in layout.shape), layout,
                         buffer=args[0]))


def _st_tensor(scope: str):
    def handler(p: _Parse, lhs, args):
        p.declare(TensorDecl(lhs, scope, parse_dtype(args[0]), p.shape(args[1])))
    return handler


def _st_copy(p: _Parse, lhs, args):
    p.emit("copy", [p.name(args[0])], [p.name(args[1])])


def _st_gemm(p: _Parse, lhs, args):
    c, a, b = (p.name(x) for x in args)
    p.emit("gemm", [a, b, c], [c])


def _st_cast(p: _Parse, lhs, args):
    src = p.decl(args[0])
    dtype = parse_dtype(args[1])
    p.declare(TensorDecl(lhs, src.scope, dtype, src.shape))
    p.emit("cast", [src.name], [lhs], cast_dtype=dtype)


def _st_rearrange(p: _Parse, lhs, args):
    src = p.decl(args[0])
    target = p.layout(args[1]) if len(args) == 2 else None
    p.declare(TensorDecl(lhs, src.scope, src.dtype, src.shape))
    p.emit("rearrange", [src.name], [lhs], rearrange_target=target)


def _st_elementwise(p: _Parse, lhs, args):
    inputs = [p.name(a) for a in args[1:]]
    first = p.tensors[inputs[0]]
    p.declare(TensorDecl(lhs, first.scope, first.dtype, first.shape))
    p.emit("elementwise", inputs, [lhs], elementwise_fn=args[0])


def _st_reduce(p: _Parse, lhs, args):
    src = p.decl(args[0])
    dim = p.int_arg(args[1], "reduce dim must be an integer")
    in_range = 0 <= dim < len(src.shape)
    p.declare(TensorDecl(lhs, src.scope, src.dtype, tuple(1 if in_range and i == dim else e
                                                          for i, e in enumerate(src.shape))))
    p.emit("reduce", [src.name], [lhs], reduce_dim=dim)


def _st_loop(p: _Parse, lhs, args):
    count = p.int_arg(args[0], "loop trip count must be an integer")
    if count < 1:
        p.fail("loop trip count must be >= 1")
    p.loops.append(count)


def _st_endloop(p: _Parse, lhs, args):
    if not p.loops:
        p.fail("endloop without matching loop")
    p.loops.pop()


def _st_annotate(p: _Parse, lhs, args):
    index = p.int_arg(args[0], "op index must be an integer")
    p.notes.append((p.line, index, p.layout(args[2])))


# head -> (lhs required?, arity predicate, usage text, handler)
_STATEMENTS: Dict[str, Tuple[bool, Callable[[list], bool], str, Callable]] = {
    "global_view": (True, lambda a: len(a) == 3, "usage: t = global_view <buffer> <dtype> <layout>",
                    _st_global_view),
    "register_tensor": (True, lambda a: len(a) == 2, "usage: t = register_tensor <dtype> <shape>",
                        _st_tensor("Register")),
    "shared_tensor": (True, lambda a: len(a) == 2, "usage: t = shared_tensor <dtype> <shape>", _st_tensor("Shared")),
    "copy": (False, lambda a: len(a) == 2, "usage: copy <src> <dst>", _st_copy),
    "gemm": (False, lambda a: len(a) == 3, "usage: gemm <c> <a> <b>", _st_gemm),
    "cast": (True, lambda a: len(a) == 2, "usage: t2 = cast <t1> <dtype>", _st_cast),
    "rearrange": (True, lambda a: len(a) in (1, 2), "usage: t2 = rearrange <t1> [<tv-layout>]", _st_rearrange),
    "elementwise": (True, lambda a: len(a) >= 2, "usage: t = elementwise <fn> <t1> ... <tn>", _st_elementwise),
    "reduce": (True, lambda a: len(a) == 2, "usage: t2 = reduce <t1> <dim>", _st_reduce),
    "loop": (False, lambda a: len(a) == 1, "usage: loop <trip-count>", _st_loop),
    "endloop": (False, lambda a: not a, "usage: endloop", _st_endloop),
    "annotate": (False, lambda a: len(a) == 3 and a[1] == "thread_arrangement",
                 "usage: annotate <op-index> thread_arrangement <layout>", _st_annotate),
}


def parse_program(text: str) -> ProgramGraph:
    """Program text -> graph (declarations resolved, loop trip counts folded into ops, op indices
    numbered in statement order, annotations attached)."""
    p = _Parse()
    lines = text.splitlines()
    for p.line, raw in enumerate(lines, start=1):
        stmt = raw.split("#", 1)[0].strip()
        if not stmt:
            continue
        lhs, _, rhs = stmt.partition("=") if "=" in stmt else (None, "", stmt)
        lhs = lhs.strip() if lhs is not None else None
        words = rhs.split()
        if not words:
            p.fail("empty statement")
        head, args = words[0], words[1:]
        spec = _STATEMENTS.get(head)
        if spec is None:
            p.fail(f"unknown statement {head!r}")
        wants_lhs, arity_ok, usage, handler = spec
        if (lhs is not None) != wants_lhs or not arity_ok(args):
            p.fail(usage)
        handler(p, lhs, args)
    if p.loops:
        raise ParseError("unterminated loop", len(lines))
    for i, op in enumerate(p.ops):
        op.index = i
    for line, index, layout in p.notes:
        if not 0 <= index < len(p.ops):
            raise ParseError(f"annotate index {index} out of range", line)
        p.ops[index].thread_arrangement = layout
    return ProgramGraph(p.tensors, p.ops)


_PRINTERS: Dict[str, Callable[[OpNode], str]] = {
    "copy": lambda op: f"copy {op.operands[0]} {op.results[0]}",
    "gemm": lambda op: f"gemm {op.operands[2]} {op.operands[0]} {op.operands[1]}",
    "cast": lambda op: f"{op.results[0]} = cast {op.operands[0]} {op.cast_dtype}",
    "rearrange": lambda op: f"{op.results[0]} = rearrange {op.operands[0]}"
                            + (f" {op.rearrange_target}" if op.rearrange_target else ""),
    "elementwise": lambda op: f"{op.results[0]} = elementwise {op.elementwise_fn} " + " ".join(op.operands),
    "reduce": lambda op: f"{op.results[0]} = reduce {op.operands[0]} {op.reduce_dim}",
}


def print_program(graph: ProgramGraph) -> str:
    """Canonical text: declarations, statements (each wrapped in its own loop), annotations."""
    derived = {r for op in graph.ops if op.kind in _DERIVED for r in op.results}
    out = []
    for t in graph.tensors.values():
        if t.scope == "Global":
            out.append(f"{t.name} = global_view {t.buffer} {t.dtype} {t.layout}")
        elif t.scope == "Shared" or t.name not in derived:
            kind = "shared_tensor" if t.scope == "Shared" else "register_tensor"
            out.append(f"{t.name} = {kind} {t.dtype} {nested.format_tuple(t.shape)}")
    for op in graph.ops:
        printer = _PRINTERS.get(op.kind)
        if printer is not None:
            stmt = printer(op)
            out.append(f"loop {op.trip_count}\n{stmt}\nendloop" if op.trip_count > 1 else stmt)
    out.extend(f"annotate {op.index} thread_arrangement {op.thread_arrangement}"
               for op in graph.ops if op.thread_arrangement is not None)
    return "\n".join(out) + "\n"


def copy_src_dst(graph: ProgramGraph, op: OpNode) -> Tuple[TensorDecl, TensorDecl]:
    if op.kind != "copy":
        raise ArityError(f"op {op.index} is not a copy")
    return graph.tensor(op.operands[0]), graph.tensor(op.results[0])


# -------------------------------------------------------------------------------------- validation
def _tensor_rules(graph: ProgramGraph) -> Iterator[str]:
    for name, t in graph.tensors.items():
        if t.dtype.bits < 8 and t.shape[0] * t.dtype.bits < 8:
            yield (f"tensor {name}: sub-byte dtype {t.dtype} needs an innermost run of >= {8 // t.dtype.bits} "
                   f"elements, got {t.shape[0]}")
        if t.scope == "Global":
            if t.layout is None:
                yield f"tensor {name}: Global tensors require a layout"
            elif any(d == 0 for e, d in t.layout.flat_modes() if e > 1):
                yield f"tensor {name}: broadcast (stride-0) global layouts unsupported"


def _check_copy(graph, op) -> Iterator[str]:
    src, dst = copy_src_dst(graph, op)
    if src.shape != dst.shape:
        yield f"op {op.index}: copy shape mismatch {src.name}{src.shape} -> {dst.name}{dst.shape}"
    if src.dtype.bits != dst.dtype.bits:
        yield f"op {op.index}: copy dtype width mismatch {src.dtype} -> {dst.dtype}"


def _check_gemm(graph, op) -> Iterator[str]:
    a, b, c = (graph.tensor(n) for n in op.operands)
    for t in (a, b, c):
        if t.scope != "Register":
            yield f"op {op.index}: gemm operand {t.name} must be Register"
        if len(t.shape) != 2:
            yield f"op {op.index}: gemm operand {t.name} must be rank-2"
    if all(len(t.shape) == 2 for t in (a, b, c)):
        (m, ka), (n, kb) = a.shape, b.shape
        if ka != kb:
            yield (f"op {op.index}: gemm reduction extent mismatch between {a.name} (K={ka}) and "
                   f"{b.name} (K={kb})")
        if tuple(c.shape) != (m, n):
            yield f"op {op.index}: gemm output extent mismatch {c.name}{c.shape} vs ({m},{n})"


def _check_register_operand(what: str):
    def rule(graph, op) -> Iterator[str]:
        if graph.tensor(op.operands[0]).scope != "Register":
            yield f"op {op.index}: {what} operand must be Register"
    return rule


def _check_reduce(graph, op) -> Iterator[str]:
    src = graph.tensor(op.operands[0])
    if op.reduce_dim is None or not 0 <= op.reduce_dim < len(src.shape):
        yield f"op {op.index}: reduce dim {op.reduce_dim} out of range for rank-{len(src.shape)} tensor {src.name}"
    yield from _check_register_operand("reduce")(graph, op)


def _check_elementwise(graph, op) -> Iterator[str]:
    shapes = {graph.tensor(n).shape for n in op.operands}
    if len(shapes) > 1:
        yield f"op {op.index}: elementwise operand shapes differ: {shapes}"


def _check_rearrange(graph, op) -> Iterator[str]:
    yield from _check_register_operand("rearrange")(graph, op)
    if op.rearrange_target is not None and op.rearrange_target.rank != 2:
        yield f"op {op.index}: rearrange target must be a two-mode (thread, value) layout"


_OP_RULES = {"copy": _check_copy, "gemm": _check_gemm, "cast": _check_register_operand("cast"),
             "reduce": _check_reduce, "elementwise": _check_elementwise, "rearrange": _check_rearrange}


def _op_rules(graph: ProgramGraph) -> Iterator[str]:
    written: set = set()
    for op in graph.ops:
        if op.kind in _DERIVED:
            yield from (f"op {op.index}: tensor {r} produced twice" for r in op.results if r in written)
        rule = _OP_RULES.get(op.kind)
        if rule is not None:
            yield from rule(graph, op)
        written.update(op.results)


def _dataflow_rules(graph: ProgramGraph) -> Iterator[str]:
    produced_by_op = {r for op in graph.ops for r in op.results}
    ready: set = set()
    for op in graph.ops:
        for name in op.operands:
            if (graph.tensor(name).scope == "Register" and name in produced_by_op and name not in ready
                    and name not in op.results):
                yield f"op {op.index}: tensor {name} used before definition"
        ready.update(op.results)


def validate(graph: ProgramGraph) -> List[str]:
    """Type / scope / shape rules; the list of diagnostics (empty = valid)."""
    return [d for rules in (_tensor_rules, _op_rules, _dataflow_rules) for d in rules(graph)]


# ------------------------------------------------------------------------------------ graph passes
def eliminate_dead_code(graph: ProgramGraph) -> ProgramGraph:
    """Keep the ops from which a copy into a Global tensor is reachable (backwards through the
    tensors they write); renumbers ``OpNode.index`` of the kept ops in place."""
    writers: Dict[str, List[OpNode]] = {}
    for op in graph.ops:
        for r in op.results:
            writers.setdefault(r, []).append(op)
    live: set = set()
    seen_tensors: set = set()
    work = deque(op for op in graph.ops if op.kind == "copy" and graph.tensor(op.results[0]).scope == "Global")
    while work:
        op = work.popleft()
        if id(op) in live:
            continue
        live.add(id(op))
        for name in op.tensors:
            if name not in seen_tensors:
                seen_tensors.add(name)
                work.extend(w for w in writers.get(name, ()) if id(w) not in live)
    kept = [op for op in graph.ops if id(op) in live]
    for i, op in enumerate(kept):
        op.index = i
    tensors = {n: d for n, d in graph.tensors.items() if n in seen_tensors or d.scope == "Global"}
    return ProgramGraph(tensors, kept, list(graph.diagnostics))


def partition_components(graph: ProgramGraph) -> List[List[OpNode]]:
    """Ops connected through Register tensors (Shared tensors cut), ordered by their first op;
    program order inside a component."""
    by_tensor: Dict[str, List[int]] = {}
    for pos, op in enumerate(graph.ops):
        for name in op.tensors:
            if graph.tensor(name).scope == "Register":
                by_tensor.setdefault(name, []).append(pos)
    component = [-1] * len(graph.ops)
    groups: List[List[int]] = []
    for start in range(len(graph.ops)):
        if component[start] >= 0:
            continue
        component[start] = len(groups)
        members, frontier = [start], deque([start])
        while frontier:
            pos = frontier.popleft()
            for name in graph.ops[pos].tensors:
                for other in by_tensor.get(name, ()):
                    if component[other] < 0:
                        component[other] = len(groups)
                        members.append(other)
                        frontier.append(other)
        groups.append(sorted(members))
    return [[graph.ops[i] for i in g] for g in groups]
