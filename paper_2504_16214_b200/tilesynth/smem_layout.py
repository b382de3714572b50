"""Shared-memory layout synthesis (paper section V).

Each copy touching a shared buffer turns its memory-side TV layout into a *layout constraint*: the
buffer's logical dimensions split into pieces whose strides are concrete (inside one thread's
vector, which must stay contiguous) or free :class:`StrideVar` s. The constraints of all copies
are unified, the free strides are materialised into a bijection, and an XOR swizzle is chosen by
the bank model. Semantics -- including which inputs fail with which error -- are the reference's
(``/root/reference/pkg/src/tilesynth/smem.py``: ``build_constraint`` ``:161-267``, ``unify``
``:282-339``, ``materialize`` ``:357-449``, ``check_tma`` ``:476-509``, ``synthesize_buffer``
``:581-647``).

Differences in the machinery: the access patterns of a copy come out of one fancy-indexing step
over the TV layout's position grid and the materialised layout's table (a ``[patterns, 32]``
address matrix), and every candidate swizzle is scored on those matrices by the vectorised bank
model (:mod:`.banking`). Materialisation is a small "stride chain" object that extends the
chain run by run.
"""
from __future__ import annotations

import itertools
import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple, Union

import numpy as np

from .banking import IDENTITY_SWIZZLE, AccessPattern, Swizzle, best_swizzle, candidate_swizzles, phase_degrees
from .errors import LayoutIncompatible, MisalignedAccess, NotInvertible, StrideConflict, Unsatisfiable
from .layout_algebra import Layout, inverse
from .tvl import TvLayout, filter_replication

_uids = itertools.count(1)


class StrideVar:
    """A free stride; its value must be a multiple of ``divisibility``."""

    __slots__ = ("uid", "divisibility")

    def __init__(self, divisibility: int = 1, uid: Optional[int] = None):
        self.uid = next(_uids) if uid is None else uid
        self.divisibility = divisibility

    def __repr__(self) -> str:
        return f"D{self.uid}"


StrideEntry = Union[int, StrideVar]
Piece = Tuple[int, StrideEntry]


def _is_free(entry) -> bool:
    return isinstance(entry, StrideVar)


@dataclass
class LayoutConstraint:
    """``splits[i]``: the (size, stride) pieces of logical dimension i, fastest first."""

    dims: Tuple[int, ...]
    splits: List[List[Piece]]

    def size(self) -> int:
        return math.prod(self.dims)

    def concrete_modes(self) -> List[Tuple[int, int]]:
        return [p for dim in self.splits for p in dim if not _is_free(p[1])]

    def render(self) -> str:
        """``(shape):(strides)`` with variables named D1, D2, ... in order of first appearance."""
        names: Dict[int, str] = {}

        def text(d):
            if not _is_free(d):
                return str(d)
            return names.setdefault(d.uid, f"D{len(names) + 1}")

        def group(items):
            return items[0] if len(items) == 1 else "(" + ",".join(items) + ")"

        shape = [group([str(s) for s, _ in dim]) for dim in self.splits]
        stride = [group([text(d) for _, d in dim]) for dim in self.splits]
        return "(" + ",".join(shape) + "):(" + ",".join(stride) + ")"

    def structure_key(self) -> Tuple:
        return tuple(tuple((s, "var" if _is_free(d) else d) for s, d in dim) for dim in self.splits)

    def __str__(self) -> str:
        return self.render()


def _split_top(text: str) -> List[str]:
    """Top-level comma-separated items of a parenthesised list."""
    if not (text.startswith("(") and text.endswith(")")):
        raise LayoutIncompatible(f"bad constraint text {text!r}")
    items, depth, start = [], 0, 1
    for i, ch in enumerate(text[1:-1], start=1):
        depth += (ch == "(") - (ch == ")")
        if ch == "," and depth == 0:
            items.append(text[start:i])
            start = i + 1
    items.append(text[start:-1])
    return items


def parse_constraint(text: str) -> LayoutConstraint:
    """``"((8,8),64):((1,D1),D2)"`` -> constraint (equal variable names share one StrideVar)."""
    shape_text, stride_text = "".join(text.split()).split(":")
    shapes, strides = _split_top(shape_text), _split_top(stride_text)
    if len(shapes) != len(strides):
        raise LayoutIncompatible("constraint shape/stride arity mismatch")
    named: Dict[str, StrideVar] = {}

    def entry(tok: str) -> StrideEntry:
        return int(tok) if tok.isdigit() else named.setdefault(tok, StrideVar())

    splits = []
    for sh, st in zip(shapes, strides):
        if sh.startswith("(") != st.startswith("("):
            raise LayoutIncompatible("constraint dim structure mismatch")
        sizes = sh[1:-1].split(",") if sh.startswith("(") else [sh]
        toks = st[1:-1].split(",") if st.startswith("(") else [st]
        splits.append([(int(a), entry(b)) for a, b in zip(sizes, toks)])
    return LayoutConstraint(tuple(math.prod(s for s, _ in dim) for dim in splits), splits)


# ------------------------------------------------------------------------------------------- build
def _cut_points(extent: int, weight: int, bounds: Sequence[int]) -> List[int]:
    """Local positions inside a run of ``extent`` steps of ``weight`` where a boundary falls."""
    out = []
    for b in bounds:
        if weight < b < weight * extent:
            if b % weight:
                raise LayoutIncompatible(f"boundary {b} misaligned with mode weight {weight}")
            out.append(b // weight)
    return out


def build_constraint(f: TvLayout, vector_elems: int, dims: Tuple[int, ...]) -> LayoutConstraint:
    """The constraint one copy puts on its buffer: every thread's ``vector_elems`` consecutive values
    must be contiguous (concrete strides), everything else is free. LayoutIncompatible when the
    (de-replicated) access is not a bijection onto the buffer."""
    f = filter_replication(f)
    total = math.prod(dims)
    if f.threads * f.values != total:
        raise LayoutIncompatible(f"access layout covers {f.threads * f.values} of {total} elements")
    try:
        back = inverse(f.layout)      # logical position -> (thread, value) index
    except NotInvertible as e:
        raise LayoutIncompatible(str(e)) from e
    vec_lo, vec_hi = f.threads, f.threads * vector_elems
    dim_ends = list(itertools.accumulate(dims, lambda a, b: a * b))
    dim_of = lambda lw: next((i for i, end in enumerate(dim_ends) if lw < end), 0)  # noqa: E731
    splits: List[List[Piece]] = [[] for _ in dims]
    logical = 1
    for extent, tv_weight in back.flat_modes():
        cuts = sorted(set(_cut_points(extent, tv_weight, (vec_lo, vec_hi)) + _cut_points(extent, logical, dim_ends)))
        prev = 1
        for point in cuts + [extent]:
            if point % prev or extent % point:
                raise LayoutIncompatible(f"cannot split mode of size {extent} at local point {point}")
            size = point // prev
            if size > 1 or (prev == 1 and point == extent):
                w = tv_weight * prev
                stride = w // f.threads if vec_lo <= w < vec_hi else StrideVar(vector_elems)
                dim = splits[dim_of(logical * prev)]
                if _is_free(stride) and dim and _is_free(dim[-1][1]):   # fuse neighbouring free pieces
                    dim[-1] = (dim[-1][0] * size, StrideVar(max(dim[-1][1].divisibility, stride.divisibility)))
                else:
                    dim.append((size, stride))
            prev = point
        logical *= extent
    return LayoutConstraint(tuple(dims), [dim or [(1, StrideVar(1))] for dim in splits])


# ------------------------------------------------------------------------------------------- unify
def _take(piece: Piece, k: int) -> Tuple[Piece, Optional[Piece]]:
    """First k positions of a piece, and the rest (None when nothing is left)."""
    size, d = piece
    if size == k:
        return piece, None
    if _is_free(d):
        return (k, StrideVar(d.divisibility)), (size // k, StrideVar(d.divisibility))
    return (k, d), (size // k, d * k)


def _meet(a: StrideEntry, b: StrideEntry) -> StrideEntry:
    if _is_free(a) and _is_free(b):
        return StrideVar(max(a.divisibility, b.divisibility))
    if not _is_free(a) and not _is_free(b) and a != b:
        raise StrideConflict(f"determined strides disagree: {a} vs {b}")
    return b if _is_free(a) else a


def _chain_check(c: LayoutConstraint) -> None:
    """Concrete pieces must nest into one prefix-product chain (no two address fields overlap)."""
    span = 1
    for size, stride in sorted(c.concrete_modes(), key=lambda m: m[1]):
        if stride < span or stride % span:
            raise StrideConflict(f"determined modes overlap: ({size}:{stride}) clashes below span {span}")
        span = stride * size


def unify(c1: LayoutConstraint, c2: LayoutConstraint) -> LayoutConstraint:
    """The least-committed constraint holding every concrete piece of both (free pieces split
    freely, concrete ones linearly); disagreements -> StrideConflict."""
    if c1.dims != c2.dims:
        raise StrideConflict(f"buffer extents differ: {c1.dims} vs {c2.dims}")
    out = []
    for xs, ys in zip(c1.splits, c2.splits):
        xs, ys, merged = list(xs), list(ys), []
        while xs and ys:
            k = min(xs[0][0], ys[0][0])
            if xs[0][0] % k or ys[0][0] % k:
                raise StrideConflict(f"dimension split sizes misalign: {xs[0][0]} vs {ys[0][0]}")
            (_, dx), rest_x = _take(xs[0], k)
            (_, dy), rest_y = _take(ys[0], k)
            xs[0:1] = [rest_x] if rest_x else []
            ys[0:1] = [rest_y] if rest_y else []
            merged.append((k, _meet(dx, dy)))
        if xs or ys:
            raise StrideConflict("dimension split sizes do not cover the dim")
        out.append(merged)
    result = LayoutConstraint(c1.dims, out)
    _chain_check(result)
    return result


# ------------------------------------------------------------------------------------- materialize
class _StrideChain:
    """Builds a bijection's stride chain: concrete pieces in stride order, free pieces (in logical
    order, split by gcd where needed) filling the gaps below them and then extending the top."""

    def __init__(self, c: LayoutConstraint):
        self.free = [[dim, pos, size, var] for dim, pieces in enumerate(c.splits)
                     for pos, (size, var) in enumerate(pieces) if _is_free(var)]
        self.placed: Dict[Tuple[int, int], List[Tuple[int, int]]] = {
            (dim, pos): [(size, d)] for dim, pieces in enumerate(c.splits)
            for pos, (size, d) in enumerate(pieces) if not _is_free(d)}
        self.top = 1

    def put(self, dim: int, pos: int, size: int) -> None:
        self.placed.setdefault((dim, pos), []).append((size, self.top))
        self.top *= size

    def fill_to(self, target: int) -> None:
        gap = target // self.top
        while gap > 1:
            hit = next(((e, math.gcd(e[2], gap)) for e in self.free
                        if math.gcd(e[2], gap) > 1 and self.top % e[3].divisibility == 0), None)
            if hit is None:
                raise Unsatisfiable(f"cannot fill stride-chain gap of {gap} at {self.top}")
            entry, g = hit
            if entry[2] > g:
                entry[2] //= g
            else:
                self.free.remove(entry)
            gap //= g
            self.put(entry[0], entry[1], g)

    def extend_with_rest(self) -> None:
        for dim, pos, size, var in self.free:
            if self.top % var.divisibility:
                raise Unsatisfiable(f"stride {self.top} violates divisibility {var.divisibility} of variable {var!r}")
            self.put(dim, pos, size)
        self.free = []


def _fuse(runs: List[Tuple[int, int]]) -> List[Tuple[int, int]]:
    out: List[Tuple[int, int]] = []
    for size, stride in runs:
        if size == 1:
            continue
        if out and stride == out[-1][0] * out[-1][1]:
            out[-1] = (out[-1][0] * size, out[-1][1])
        else:
            out.append((size, stride))
    return out or [(1, 0)]


def materialize(c: LayoutConstraint) -> Layout:
    """Assign the free strides so the constraint becomes a bijection onto [0, size)."""
    _chain_check(c)
    chain = _StrideChain(c)
    for size, stride in sorted(c.concrete_modes(), key=lambda m: m[1]):
        if stride > chain.top:
            chain.fill_to(stride)
        chain.top = stride * size
    chain.extend_with_rest()
    if chain.top != c.size():
        raise Unsatisfiable(f"materialized span {chain.top} != buffer size {c.size()}")
    shapes, strides = [], []
    for dim, pieces in enumerate(c.splits):
        runs = [r for pos in range(len(pieces)) for r in sorted(chain.placed[(dim, pos)], key=lambda r: r[1])]
        fused = _fuse(runs)
        shapes.append(fused[0][0] if len(fused) == 1 else tuple(s for s, _ in fused))
        strides.append(fused[0][1] if len(fused) == 1 else tuple(d for _, d in fused))
    return Layout(tuple(shapes), tuple(strides))


# ------------------------------------------------------------------------------------------- TMA
@dataclass
class TmaCheck:
    feasible: bool
    reason: str = ""
    hint: Optional[Layout] = None


def check_tma(c: LayoutConstraint, element_bits: int, *, max_dims: int = 5, align_bytes: int = 16,
              max_box: int = 256) -> TmaCheck:
    """Can a bulk-copy (TMA) engine serve this buffer? Few enough box dimensions, every extent within
    the box cap, and a contiguous innermost run of at least ``align_bytes``; the hint is the
    materialised layout."""
    n_modes = sum(len(dim) for dim in c.splits)
    if n_modes > max_dims:
        return TmaCheck(False, f"{n_modes} dims exceed limit {max_dims}")
    if max(c.dims) > max_box:
        return TmaCheck(False, f"extent exceeds box cap {max_box}")
    run = 1
    for size, stride in sorted(c.concrete_modes(), key=lambda m: m[1]):
        if stride == run:
            run *= size
    if run * element_bits // 8 < align_bytes:
        return TmaCheck(False, f"innermost contiguous run is {run * element_bits // 8}B < {align_bytes}B")
    try:
        return TmaCheck(True, "", materialize(c))
    except Unsatisfiable as e:
        return TmaCheck(False, str(e))


# ----------------------------------------------------------------------------------------- buffers
@dataclass
class BufferCopy:
    """One copy touching a shared buffer: its memory-side TV layout, vector width, instruction."""

    op_index: int
    access: TvLayout
    vector_elems: int
    instruction: str


@dataclass
class SmemLayout:
    buffer: str
    layout: Layout
    swizzle: Swizzle
    element_bits: int
    copy_conflicts: Dict[int, int] = field(default_factory=dict)
    identity_conflicts: Dict[int, int] = field(default_factory=dict)
    constraint: Optional[LayoutConstraint] = None
    copies: List[BufferCopy] = field(default_factory=list)

    def byte_address(self, logical: int) -> int:
        return self.swizzle(self.layout(logical) * self.element_bits // 8)

    def render(self) -> str:
        return f"{self.layout} (+) {self.swizzle}"


def _access_width(copy: BufferCopy, element_bits: int) -> int:
    return max(1, copy.vector_elems * element_bits // 8)


def pattern_matrix(m: Layout, element_bits: int, copy: BufferCopy) -> np.ndarray:
    """Pre-swizzle byte addresses ``[patterns, lanes]``: one row per (warp, vector iteration) in that
    order, first occurrences only. Raises MisalignedAccess like constructing the patterns would."""
    f = copy.access
    v = copy.vector_elems
    width = _access_width(copy, element_bits)
    lanes = min(32, f.threads)
    warps = max(1, f.threads // 32)
    iters = max(1, f.values // v)
    grid = f.grid()[: warps * lanes, np.arange(iters) * v]                 # [threads, iters]
    addrs = m.table()[grid] * element_bits // 8
    addrs = addrs.reshape(warps, lanes, iters).transpose(0, 2, 1).reshape(warps * iters, lanes)
    if width not in (1, 2, 4, 8, 16):
        raise MisalignedAccess(f"unsupported access width {width}")
    bad = addrs % width != 0
    if bad.any():
        raise MisalignedAccess(f"address {int(addrs.reshape(-1)[np.argmax(bad.reshape(-1))])} "
                               f"not aligned to width {width}")
    _, first = np.unique(addrs, axis=0, return_index=True)
    return addrs[np.sort(first)]


def access_patterns(m: Layout, element_bits: int, copy: BufferCopy) -> List[AccessPattern]:
    """The copy's distinct warp-wide access patterns (pre-swizzle byte addresses)."""
    width = _access_width(copy, element_bits)
    return [AccessPattern(tuple(int(a) for a in row), width) for row in pattern_matrix(m, element_bits, copy)]


_BUFFER_CACHE: Dict[Tuple, SmemLayout] = {}


def synthesize_buffer(buffer: str, dims: Tuple[int, ...], element_bits: int,
                      copies: Sequence[BufferCopy]) -> SmemLayout:
    """Unify the copies' constraints, materialise, pick a swizzle. Memoised on (extents, element
    width, per-copy (op, access layout, tile, vector)) for the life of the process."""
    if not copies:
        raise Unsatisfiable(f"buffer {buffer} has no copies")
    key = (dims, element_bits, tuple((c.op_index, str(c.access.layout), c.access.tile, c.vector_elems)
                                     for c in copies))
    hit = _BUFFER_CACHE.get(key)
    if hit is not None:
        return SmemLayout(buffer, hit.layout, hit.swizzle, hit.element_bits, dict(hit.copy_conflicts),
                          dict(hit.identity_conflicts), hit.constraint, list(hit.copies))
    constraint = build_constraint(copies[0].access, copies[0].vector_elems, dims)
    for c in copies[1:]:
        constraint = unify(constraint, build_constraint(c.access, c.vector_elems, dims))
    m = materialize(constraint)
    widest = max(_access_width(c, element_bits) for c in copies)
    sets = [(pattern_matrix(m, element_bits, c), _access_width(c, element_bits)) for c in copies]
    best, _, degrees = best_swizzle(sets, candidate_swizzles(min_base=max(2, (widest - 1).bit_length())))
    result = SmemLayout(buffer, m, best, element_bits, constraint=constraint, copies=list(copies))
    for c, d, (addrs, width) in zip(copies, degrees, sets):
        result.copy_conflicts[c.op_index] = int(d.max())
        result.identity_conflicts[c.op_index] = int(phase_degrees(addrs, width).max())
    _BUFFER_CACHE[key] = result
    return result
