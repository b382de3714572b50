"""Integer layouts ``shape : stride`` and their algebra.

A :class:`Layout` maps a (colex-decomposed) index to ``sum(digit * stride)`` over the leaves of its
shape tree. Behaviour -- results, mode structure of results, error classes -- follows the reference
(``/root/reference/pkg/src/tilesynth/layout.py:32-505``); the representation does not:

* a layout keeps its leaves as a flat tuple of ``(extent, stride)`` runs next to the nested
  tuples, so evaluation is one ``divmod`` chain and never recurses for linear indices;
* :meth:`Layout.table` materialises the whole map as a numpy vector (outer sums, one per run) --
  the shared-memory / bank-conflict passes index it instead of evaluating point by point;
* the pure operations (coalesce, compose, inverse) are memoised on the immutable operands, which
  the candidate search re-issues with the same arguments thousands of times.
"""
from __future__ import annotations

import functools
import math
from typing import List, Sequence, Tuple, Union

import numpy as np

from . import nested
from .errors import (LayoutIncompatible, NotComplementable, NotDivisible, NotInvertible, OutOfDomain, ParseError,
                     ShapeMismatch)
from .nested import IntTuple

Coord = Union[int, Tuple["Coord", ...]]
Run = Tuple[int, int]


class Layout:
    """Immutable ``shape : stride`` function; the top level is always a tuple of modes."""

    __slots__ = ("shape", "stride", "_runs", "_size", "_hash", "_table")

    def __init__(self, shape: IntTuple, stride: IntTuple):
        shape = (shape,) if isinstance(shape, int) else shape
        stride = (stride,) if isinstance(stride, int) else stride
        nested.validate(shape, min_leaf=1)
        nested.validate(stride, min_leaf=0)
        if not nested.congruent(shape, stride):
            raise ShapeMismatch(f"shape {nested.format_tuple(shape)} and stride "
                                f"{nested.format_tuple(stride)} are not congruent")
        runs = tuple(zip(nested.leaves(shape), nested.leaves(stride)))
        for name, value in (("shape", shape), ("stride", stride), ("_runs", runs),
                            ("_size", math.prod(e for e, _ in runs)), ("_hash", None), ("_table", None)):
            object.__setattr__(self, name, value)

    def __setattr__(self, name, value):
        raise AttributeError("Layout is immutable")

    # -- structure -------------------------------------------------------------------------
    @property
    def rank(self) -> int:
        return len(self.shape)

    def size(self) -> int:
        return self._size

    def cosize(self) -> int:
        return 1 + sum((e - 1) * d for e, d in self._runs)

    def mode(self, i: int) -> "Layout":
        return Layout(self.shape[i], self.stride[i])

    def modes(self) -> List["Layout"]:
        return [self.mode(i) for i in range(len(self.shape))]

    def flat_modes(self) -> List[Run]:
        return list(self._runs)

    # -- evaluation ------------------------------------------------------------------------
    def __call__(self, x: Coord) -> int:
        if isinstance(x, int):
            return _linear(self._runs, self._size, x)
        return _at_coord(self.shape, self.stride, x)

    def map(self) -> List[int]:
        return self.table().tolist()

    def table(self) -> np.ndarray:
        """All values as an int64 vector indexed by the linear index (cached)."""
        if self._table is None:
            acc = np.zeros(1, dtype=np.int64)
            for extent, stride in self._runs:
                acc = (np.arange(extent, dtype=np.int64)[:, None] * stride + acc[None, :]).reshape(-1)
            acc.setflags(write=False)
            object.__setattr__(self, "_table", acc)
        return self._table

    # -- identity --------------------------------------------------------------------------
    def __eq__(self, other) -> bool:
        return isinstance(other, Layout) and self.shape == other.shape and self.stride == other.stride

    def __hash__(self) -> int:
        if self._hash is None:
            object.__setattr__(self, "_hash", hash((self.shape, self.stride)))
        return self._hash

    def equivalent(self, other: "Layout") -> bool:
        """Same function (compared through the coalesced forms)."""
        return coalesce(self) == coalesce(other)

    def __str__(self) -> str:
        return nested.format_tuple(self.shape) + ":" + nested.format_tuple(self.stride)

    def __repr__(self) -> str:
        return f"Layout({self})"

    def __reduce__(self):
        return Layout, (self.shape, self.stride)


def _linear(runs, total: int, x: int) -> int:
    if x < 0 or x >= total:
        raise OutOfDomain(f"index {x} outside [0, {total})")
    value = 0
    for extent, stride in runs:
        x, digit = divmod(x, extent)
        value += digit * stride
    return value


def _at_coord(shape, stride, coord) -> int:
    """Evaluate at a (possibly partial) coordinate tree; an int at a tuple node is a linear index
    into that subtree."""
    value = 0
    work = [(shape, stride, coord)]
    while work:
        s, d, c = work.pop()
        if isinstance(s, int):
            if not isinstance(c, int):
                raise ShapeMismatch(f"tuple coordinate for scalar shape {s}")
            if not 0 <= c < s:
                raise OutOfDomain(f"coordinate {c} outside [0, {s})")
            value += c * d
        elif isinstance(c, int):
            runs = tuple(zip(nested.leaves(s), nested.leaves(d)))
            value += _linear(runs, math.prod(e for e, _ in runs), c)
        elif len(c) != len(s):
            raise ShapeMismatch(f"coordinate arity {len(c)} != mode count {len(s)}")
        else:
            work.extend(zip(s, d, c))
    return value


def identity_layout(n: int) -> Layout:
    return Layout((n,), (1,))


def parse_layout(text: str) -> Layout:
    """``"((2,4),(2,2)):((8,1),(4,16))"`` -> Layout (whitespace ignored)."""
    body = "".join(text.split())
    parts = body.split(":")
    if len(parts) != 2:
        raise ParseError(f"layout needs exactly one ':': {text!r}")
    return Layout(nested.parse_tuple(parts[0]), nested.parse_tuple(parts[1]))


def _from_runs(runs: Sequence[Run]) -> Layout:
    """Flat layout from runs; no runs -> the unit layout ``(1):(0)``."""
    if not runs:
        return Layout((1,), (0,))
    return Layout(tuple(e for e, _ in runs), tuple(d for _, d in runs))


def _merged(runs) -> List[Run]:
    """Drop extent-1 runs and fuse a run into its predecessor when it continues it."""
    out: List[Run] = []
    for extent, stride in runs:
        if extent == 1:
            continue
        if out and out[-1][0] * out[-1][1] == stride:
            out[-1] = (out[-1][0] * extent, out[-1][1])
        else:
            out.append((extent, stride))
    return out


@functools.lru_cache(maxsize=1 << 16)
def coalesce(layout: Layout) -> Layout:
    """Pointwise-equal flat form with mergeable neighbours fused and unit runs dropped."""
    return _from_runs(_merged(layout._runs))


# -------------------------------------------------------------------------------------- compose
def _div_or_one(a: int, b: int) -> int:
    """a / b when b divides a; 1 when a divides b; otherwise the operands are incompatible."""
    if b and a % b == 0:
        return a // b
    if a and b % a == 0:
        return 1
    raise LayoutIncompatible(f"divisibility condition violated: {a} vs {b}")


def _image_of_run(base: Sequence[Run], extent: int, step: int) -> List[Run]:
    """The runs that ``x -> base(step * x)``, x < extent, traces through a flat (coalesced) base."""
    if extent == 1:
        return []
    if step == 0:
        return [(extent, 0)]
    pieces: List[Run] = []
    left, stride = extent, step
    *inner, (_, last_stride) = base
    for mode_extent, mode_stride in inner:
        if left == 1:
            break
        fits = _div_or_one(mode_extent, stride)   # steps of `stride` inside this base mode
        take = fits if fits < left else left
        if take > 1:
            pieces.append((take, mode_stride * stride))
        left, stride = _div_or_one(left, fits), _div_or_one(stride, mode_extent)
    if left > 1:
        pieces.append((left, last_stride * stride))
    return pieces


@functools.lru_cache(maxsize=1 << 16)
def compose(a: Layout, b: Layout) -> Layout:
    """``(a o b)(x) = a(b(x))``; the result has b's mode tree, each leaf of b expanded into the runs
    its image traces through a (b's image must lie inside a's domain)."""
    if b.cosize() > a.size():
        raise OutOfDomain(f"image of {b} (cosize {b.cosize()}) escapes domain of {a} (size {a.size()})")
    base = coalesce(a)._runs

    def build(s, d):
        shapes, strides = [], []
        for sub_s, sub_d in zip(s, d):
            if isinstance(sub_s, tuple):
                ts, td = build(sub_s, sub_d)
                shapes.append(ts)
                strides.append(td)
            else:
                for piece in _image_of_run(base, sub_s, sub_d):
                    shapes.append(piece[0])
                    strides.append(piece[1])
        return (tuple(shapes), tuple(strides)) if shapes else ((1,), (0,))

    return Layout(*build(b.shape, b.stride))


# ------------------------------------------------------------------------- complement / inverse
def complement(a: Layout, codomain_size: int) -> Layout:
    """Layout c with concat(a, c) a bijection onto [0, codomain_size)."""
    runs = sorted((r for r in coalesce(a)._runs if r[0] > 1), key=lambda r: r[1])
    if any(d == 0 for _, d in runs):
        raise NotComplementable("layout with stride-0 mode is not injective")
    gaps: List[Run] = []
    span = 1
    for extent, stride in runs:
        if stride < span or stride % span:
            raise NotComplementable(f"mode ({extent}:{stride}) overlaps already-covered span {span}")
        if stride > span:
            gaps.append((stride // span, span))
        span = stride * extent
    if codomain_size % span:
        raise NotComplementable(f"codomain {codomain_size} incompatible with span {span}")
    if codomain_size > span:
        gaps.append((codomain_size // span, span))
    return _from_runs(_merged(gaps))


@functools.lru_cache(maxsize=1 << 16)
def inverse(a: Layout) -> Layout:
    """Inverse of a bijection onto [0, size): sorting the runs by stride must give an exact chain
    of prefix products; the result is flat and coalesced."""
    runs = [r for r in coalesce(a)._runs if r[0] > 1]
    if any(d == 0 for _, d in runs):
        raise NotInvertible("stride-0 mode with extent > 1 is not injective")
    weights = np.cumprod([1] + [e for e, _ in runs])[:-1].tolist()
    chain: List[Run] = []
    expect = 1
    for idx in sorted(range(len(runs)), key=lambda i: runs[i][1]):
        extent, stride = runs[idx]
        if stride != expect:
            raise NotInvertible(f"sorted strides of {a} do not form exact prefix products")
        chain.append((extent, int(weights[idx])))
        expect *= extent
    return _from_runs(_merged(chain))


def concat(a: Layout, b: Layout) -> Layout:
    """``concat(a, b)((x, y)) = a(x) + b(y)``."""
    return Layout((a.shape, b.shape), (a.stride, b.stride))


# --------------------------------------------------------------------------------- restriction
def _packed(runs: Sequence[Run]):
    """One mode from its runs: a single run is a scalar pair, several a tuple pair."""
    if len(runs) == 1:
        return runs[0]
    return tuple(e for e, _ in runs), tuple(d for _, d in runs)


def _cut(runs: Sequence[Run], n: int, total: int):
    """Split runs (colex) at index-space size n -> (first n positions' runs, the remainder)."""
    head: List[Run] = []
    tail: List[Run] = []
    have = 1
    for extent, stride in runs:
        if have == n:
            tail.append((extent, stride))
        elif have * extent <= n:
            head.append((extent, stride))
            have *= extent
        else:  # the boundary falls inside this run
            if n % have:
                raise NotDivisible(f"restriction size {n} misaligned at {have}")
            part = n // have
            if extent % part:
                raise NotDivisible(f"leaf of size {extent} not divisible by required factor {part}")
            if part > 1:
                head.append((part, stride))
            tail.append((extent // part, stride * part))
            have = n
    if have != n:
        raise NotDivisible(f"mode of size {total} cannot reach restriction size {n}")
    return head or [(1, 0)], tail


def restrict_mode_split(a: Layout, mode_index: int, n: int) -> Tuple[Layout, List[Run]]:
    """Keep the colex-fastest n positions of one top-level mode; also return the dropped runs."""
    if not 0 <= mode_index < a.rank:
        raise ShapeMismatch(f"mode index {mode_index} out of range")
    runs = a.mode(mode_index)._runs
    total = math.prod(e for e, _ in runs)
    if n < 1 or n > total:
        raise NotDivisible(f"cannot restrict mode of size {total} to {n}")
    if n == total:
        return a, []
    kept, dropped = _cut(runs, n, total)
    s, d = _packed(kept)
    shape = a.shape[:mode_index] + (s,) + a.shape[mode_index + 1:]
    stride = a.stride[:mode_index] + (d,) + a.stride[mode_index + 1:]
    return Layout(shape, stride), dropped


def restrict_mode(a: Layout, mode_index: int, n: int) -> Layout:
    return restrict_mode_split(a, mode_index, n)[0]


def restrict_first_mode(a: Layout, n: int) -> Layout:
    return restrict_mode_split(a, 0, n)[0]


def group_modes(a: Layout, sizes: Sequence[int]) -> Layout:
    """Re-split a layout's runs (colex) into top-level modes of the given sizes."""
    pending = list(a._runs)
    shapes, strides = [], []
    for want in sizes:
        took: List[Run] = []
        have = 1
        while have < want:
            if not pending:
                raise NotDivisible(f"layout of size {a.size()} cannot group into {tuple(sizes)}")
            extent, stride = pending[0]
            if have * extent <= want:
                took.append(pending.pop(0))
                have *= extent
                continue
            part = want // have
            if want % have or extent % part:
                raise NotDivisible(f"group boundary {want} misaligned inside a leaf of {extent}")
            took.append((part, stride))
            pending[0] = (extent // part, stride * part)
            have = want
        s, d = _packed(took or [(1, 0)])
        shapes.append(s)
        strides.append(d)
    if any(extent != 1 for extent, _ in pending):
        raise NotDivisible(f"layout of size {a.size()} does not cover groups {tuple(sizes)}")
    return Layout(tuple(shapes), tuple(strides))


# ------------------------------------------------------------------------------ 2-D dimension maps
def projection_layout(extents: Tuple[int, int], out_dim: int) -> Layout:
    """Colex linear index over ``extents`` -> its ``out_dim`` coordinate."""
    return Layout(tuple(extents), (1, 0) if out_dim == 0 else (0, 1))


def embedding_layout(extents: Tuple[int, int], in_dim: int) -> Layout:
    """1-D coordinate along ``in_dim`` -> linear index with the other coordinate 0."""
    return Layout((extents[in_dim],), (1 if in_dim == 0 else extents[0],))


def dim_restrict(composite: Layout, in_dim: int, out_dim: int, in_extents: Tuple[int, int],
                 out_extents: Tuple[int, int]) -> Layout:
    """The 1-D map (input coordinate along in_dim, other one 0) -> output coordinate out_dim of a
    2-D tile -> 2-D tensor mapping (Theorem-1 equations of the report's explain trace)."""
    if len(in_extents) != 2 or len(out_extents) != 2:
        raise ShapeMismatch("dim_restrict expects 2-D extents")
    if composite.rank != 2:
        raise ShapeMismatch("composite must have exactly two modes")
    sizes = tuple(nested.size(s) for s in composite.shape)
    if sizes != tuple(in_extents):
        raise ShapeMismatch(f"composite mode sizes {sizes} != input extents {in_extents}")
    inner = compose(composite, embedding_layout(tuple(in_extents), in_dim))
    return coalesce(compose(projection_layout(tuple(out_extents), out_dim), inner))
