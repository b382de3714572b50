"""Shared-memory layout synthesis: per-copy layout constraints, their unification, materialisation
into a bijective buffer layout, the TMA feasibility check, and the swizzle choice.

Contract: /root/reference/pkg/src/tilesynth/smem.py:1-647 (constraint text, unify / materialize
results and error classes, check_tma, synthesize_buffer's layout, swizzle and per-copy conflicts).

Construction here:

* A constraint dimension is a *factorisation*: a list of ``(extent, entry)`` pieces whose extents
  multiply to the dimension; an entry is a concrete stride (int) or a :class:`StrideVar`.
* :func:`build_constraint` inverts the (de-duplicated) access map and cuts its runs at two sets of
  boundaries at once -- the vector field [T, T*vec) in thread-value index space and the dimension
  ends in logical space -- with one generic :func:`_refine` over "boundary lists".
* :func:`unify` overlays two factorisations of each dimension on the cumulative-extent axis: two
  cursors walk the piece ends, each step ends at the nearer one, and the piece of the common
  refinement takes its entry from the piece of each side that contains it.
* :func:`materialize` runs a stride-chain cursor: concrete pieces pin the chain, free pieces fill
  the gaps (first fitting piece in logical order, split by gcd) and then extend the chain.
* The swizzle search builds every copy's warp address matrix straight from the buffer layout's
  table and the access grid (numpy fancy indexing) and scores all candidate swizzles at once
  (:func:`score_pattern_matrix`).

The first part of the module is the bank model (contract /root/reference/pkg/src/tilesynth/swizzle.py:
1-160: the swizzle family; 32 banks x 4 B; an 8-byte access runs in 2 phases of 16 threads, a
16-byte access in 4 phases of 8; a phase's degree is the largest number of distinct words one bank
serves; the least total over the patterns wins, ties toward smaller (bits, base, shift), swizzles
that would split a vector are ineligible). It is evaluated on whole arrays: a batch of warp-wide
access patterns (rows of an int64 matrix) against every candidate swizzle at once, so a buffer's
swizzle search is one numpy pass (:func:`score_pattern_matrix`) instead of a Python loop per
(swizzle, pattern, lane).
"""
from __future__ import annotations

import dataclasses
import math
import re
from typing import Callable, Dict, Iterable, List, Optional, Tuple, Union

import numpy as np

from .algebra import Layout, TvLayout, filter_replication, fuse_runs, inverse
from .errors import LayoutIncompatible, MisalignedAccess, NotInvertible, StrideConflict, Unsatisfiable
from .records import record

NUM_BANKS = 32
BANK_BYTES = 4
VALID_WIDTHS = (1, 2, 4, 8, 16)


class Swizzle(tuple):
    """``addr ^ (((addr >> (base + shift)) & (2^bits - 1)) << base)``; ``bits == 0`` is the identity.

    A (bits, base, shift) triple, ordered and hashed as one; ``shift >= bits`` keeps the source
    field clear of the target field."""

    __slots__ = ()

    def __new__(cls, bits, base, shift):
        if bits < 0 or base < 0:
            raise ValueError("swizzle fields are non-negative")
        if bits > 0 and shift < bits:
            raise ValueError(f"source field (shift {shift}) overlaps the {bits} target bits")
        return super().__new__(cls, (bits, base, shift))

    bits = property(lambda self: self[0])
    base = property(lambda self: self[1])
    shift = property(lambda self: self[2])

    @property
    def is_identity(self):
        return self[0] == 0

    def __call__(self, addr):
        """Swizzle one address (int) or an array of them."""
        bits, base, shift = self
        if np.ndim(addr) == 0:
            if addr < 0:
                raise ValueError("swizzle expects a non-negative address")
            return addr if not bits else addr ^ (((addr >> (base + shift)) & ((1 << bits) - 1)) << base)
        return addr ^ (((addr >> (base + shift)) & ((1 << bits) - 1)) << base) if bits else addr

    def __repr__(self):
        return "Swizzle(bits={}, base={}, shift={})".format(*self)

    def __str__(self):
        return "SW({},{},{})".format(*self)


IDENTITY_SWIZZLE = Swizzle(0, 4, 3)


class AccessPattern:
    """The byte addresses one warp-wide access issues (one per thread) and its width."""

    __slots__ = ("addresses", "width")

    def __init__(self, addresses, width):
        if width not in VALID_WIDTHS:
            raise MisalignedAccess(f"{width}-byte accesses are not modelled")
        addresses = tuple(addresses)
        if any(a % width for a in addresses):
            raise MisalignedAccess(f"an address of {addresses} is not {width}-byte aligned")
        self.addresses, self.width = addresses, width

    def __eq__(self, other):
        return isinstance(other, AccessPattern) and (self.addresses, self.width) == (other.addresses, other.width)

    def __hash__(self):
        return hash((self.addresses, self.width))

    def __repr__(self):
        return f"AccessPattern(addresses={self.addresses!r}, width={self.width})"


PatternGenerator = Callable[[Swizzle], Iterable[AccessPattern]]


# ----------------------------------------------------------------------------------------
# shared-memory layout constraints
class StrideVar:
    """A stride still to be chosen; its value must be a multiple of ``divisibility``."""

    __slots__ = ("divisibility",)

    def __init__(self, divisibility=1):
        self.divisibility = divisibility

    def __repr__(self):
        return f"StrideVar(div={self.divisibility})"


Entry = Union[int, StrideVar]
Piece = Tuple[int, Entry]


def _constraint_render(c):
    """``(s0,(s1,s2)):(1,(D1,D2))`` -- free strides numbered by first appearance."""
    names = {}

    def word(st):
        return str(st) if isinstance(st, int) else names.setdefault(id(st), f"D{len(names) + 1}")

    def group(items):
        return items[0] if len(items) == 1 else "(" + ",".join(items) + ")"

    shapes = [group([str(e) for e, _ in dim]) for dim in c.splits]
    strides = [group([word(st) for _, st in dim]) for dim in c.splits]
    return "(" + ",".join(shapes) + "):(" + ",".join(strides) + ")"


LayoutConstraint = record(
    "LayoutConstraint", ["dims", "splits"],
    "``splits[i]``: the pieces (extent, stride | StrideVar) of dimension i, fastest first; extents multiply "
    "to ``dims[i]``.", module=__name__,
    size=lambda c: math.prod(c.dims),
    concrete_modes=lambda c: [(e, st) for dim in c.splits for e, st in dim if isinstance(st, int)],
    render=_constraint_render,
    structure_key=lambda c: tuple(tuple((e, st if isinstance(st, int) else "var") for e, st in dim)
                                  for dim in c.splits),
    __str__=_constraint_render)


_ITEM = re.compile(r"\(([^()]*)\)|([^,()]+)")


# ------------------------------------------------------------------------------------- materialize
class _StrideChain:
    """The address chain of a buffer being materialised: a cursor ``reach`` (the span covered so
    far), the free pieces still to place (logical order, mutable remaining extents) and the strides
    given to every (dimension, piece) slot."""

    def __init__(self, c):
        self.c = c
        self.reach = 1
        self.slots = {}
        self.free = []
        for d, dim in enumerate(c.splits):
            for p, (e, s) in enumerate(dim):
                if isinstance(s, int):
                    self.slots[(d, p)] = [(e, s)]
                else:
                    self.free.append([d, p, e, s])

    def give(self, rec, extent, stride):
        self.slots.setdefault((rec[0], rec[1]), []).append((extent, stride))

    def close_gap(self, upto):
        """Free pieces (first fitting one in logical order, cut by gcd) until the chain reaches the
        next concrete stride ``upto``."""
        gap, at = upto // self.reach, self.reach
        while gap > 1:
            rec = next((r for r in self.free if math.gcd(r[2], gap) > 1 and at % r[3].divisibility == 0), None)
            if rec is None:
                raise Unsatisfiable(f"no free piece fits the stride gap {gap} at {at}")
            g = math.gcd(rec[2], gap)
            self.give(rec, g, at)
            rec[2] //= g
            if rec[2] == 1:
                self.free.remove(rec)
            at, gap = at * g, gap // g

    def extend(self):
        """The remaining free pieces, in logical order, on top of the chain."""
        for rec in self.free:
            if self.reach % rec[3].divisibility:
                raise Unsatisfiable(f"stride {self.reach} is not a multiple of {rec[3].divisibility}")
            self.give(rec, rec[2], self.reach)
            self.reach *= rec[2]

    def layout(self):
        dims = []
        for d, dim in enumerate(self.c.splits):
            runs = fuse_runs(r for p in range(len(dim)) for r in sorted(self.slots[(d, p)], key=lambda r: r[1]))
            runs = runs or [(1, 0)]
            dims.append(runs[0] if len(runs) == 1 else (tuple(e for e, _ in runs), tuple(st for _, st in runs)))
        return Layout(tuple(x for x, _ in dims), tuple(y for _, y in dims))


# ----------------------------------------------------------------------------------------------- TMA
TmaCheck = record("TmaCheck", ["feasible", ("reason", ""), ("hint", None)],
                  "Bulk-tensor-engine feasibility of a buffer, why not, and the materialised hint.", module=__name__)


# ------------------------------------------------------------------------------------------ buffers
BufferCopy = record(
    "BufferCopy", ["op_index", "access", "vector_elems", "instruction"],
    "One copy touching a shared buffer: its memory-side access layout, vector width (elements) and "
    "instruction name.", module=__name__)

SmemLayout = record(
    "SmemLayout", ["buffer", "layout", "swizzle", "element_bits", ("copy_conflicts", dict),
                   ("identity_conflicts", dict), ("constraint", None), ("copies", list)],
    "A synthesized shared buffer: layout, swizzle, per-copy conflict degree (chosen / identity swizzle).",
    module=__name__,
    byte_address=lambda b, logical: b.swizzle(b.layout(logical) * b.element_bits // 8),
    render=lambda b: f"{b.layout} (+) {b.swizzle}")


_MEMO: Dict[Tuple, SmemLayout] = {}


def synthesize_buffer(buffer, dims, element_bits, copies):
    """Unify the copies' constraints, materialise the layout, choose the swizzle, record each copy's
    conflict degree under it and under the identity. Memoised on (extents, width, accesses)."""
    if not copies:
        raise Unsatisfiable(f"buffer {buffer} has no copies")
    key = (tuple(dims), element_bits,
           tuple((c.op_index, c.access.layout, c.access.tile, c.vector_elems) for c in copies))
    hit = _MEMO.get(key)
    if hit is None:
        constraint = build_constraint(copies[0].access, copies[0].vector_elems, dims)
        for c in copies[1:]:
            constraint = unify(constraint, build_constraint(c.access, c.vector_elems, dims))
        m = materialize(constraint)
        widest = max(max(1, c.vector_elems * element_bits // 8) for c in copies)
        pool = candidate_swizzles(min_base=max(2, (widest - 1).bit_length()))
        groups = [warp_address_matrix(m, element_bits, c) for c in copies]
        best, _, _ = score_pattern_matrix(groups, pool)
        hit = SmemLayout(buffer, m, best, element_bits, constraint=constraint, copies=list(copies))
        for c, (rows, width) in zip(copies, groups):
            for sw, table in ((best, hit.copy_conflicts), (IDENTITY_SWIZZLE, hit.identity_conflicts)):
                table[c.op_index] = int(phase_degrees(sw(rows), width).max(initial=1))
        _MEMO[key] = hit
    return dataclasses.replace(hit, buffer=buffer, copy_conflicts=dict(hit.copy_conflicts),
                               identity_conflicts=dict(hit.identity_conflicts), copies=list(hit.copies))


def access_patterns(m, element_bits, copy):
    """The copy's distinct warp-wide accesses as :class:`AccessPattern` objects (diagnostics)."""
    rows, width = warp_address_matrix(m, element_bits, copy)
    return [AccessPattern(tuple(int(a) for a in row), width) for row in rows]


def warp_address_matrix(m, element_bits, copy):
    """Pre-swizzle byte addresses of every distinct warp-wide access of one copy: row (warp w,
    vector j) holds lane l's address of ``m(access(32 w + l, j * vec))``. Returns (rows, width)."""
    f, vec = copy.access, copy.vector_elems
    width = max(1, vec * element_bits // 8)
    if width not in VALID_WIDTHS:
        raise MisalignedAccess(f"{width}-byte accesses are not modelled")
    lanes = min(32, f.threads)
    warps = max(1, f.threads // 32)
    iters = max(1, f.values // vec)
    grid = f.grid()
    threads = (np.arange(warps)[:, None] * 32 + np.arange(lanes)).ravel()
    elems = grid[threads][:, np.arange(iters) * vec]            # [warps * lanes, iters]
    addrs = m.table()[elems] * element_bits // 8
    rows = addrs.reshape(warps, lanes, iters).transpose(0, 2, 1).reshape(-1, lanes)
    if (rows % width).any():
        raise MisalignedAccess(f"a {width}-byte access of copy {copy.op_index} is misaligned")
    return np.unique(rows, axis=0), width


def materialize(c):
    """Pick the free strides so the layout is a bijection onto [0, size): concrete pieces first by
    stride, free pieces fill the chain gaps and then extend the chain in logical order."""
    _check_chain(c)
    chain = _StrideChain(c)
    for e, s in sorted(c.concrete_modes(), key=lambda m: m[1]):
        if s > chain.reach:
            chain.close_gap(s)
        chain.reach = s * e
    chain.extend()
    if chain.reach != c.size():
        raise Unsatisfiable(f"the strides span {chain.reach}, the buffer holds {c.size()}")
    return chain.layout()


def unify(c1, c2):
    """Least-committed constraint holding every concrete stride of both. StrideConflict when the
    factorisations cannot be overlaid, concrete strides disagree, or the concrete pieces overlap."""
    if c1.dims != c2.dims:
        raise StrideConflict(f"buffer extents {c1.dims} and {c2.dims} differ")
    merged = []
    for xs, ys in zip(c1.splits, c2.splits):
        bx, by = _bounds(xs), _bounds(ys)
        dim, lo, i, j = [], 1, 0, 0
        while i < len(bx) and j < len(by):
            hi = min(bx[i][1], by[j][1])      # next boundary of the common refinement
            if bx[i][1] % hi or by[j][1] % hi:
                raise StrideConflict(f"piece boundaries misalign at {hi}")
            a, b = _sub_entry(bx[i], lo), _sub_entry(by[j], lo)
            if isinstance(a, int) and isinstance(b, int) and a != b:
                raise StrideConflict(f"concrete strides {a} and {b} disagree")
            if isinstance(a, int) or isinstance(b, int):
                dim.append((hi // lo, a if isinstance(a, int) else b))
            else:
                dim.append((hi // lo, StrideVar(max(a.divisibility, b.divisibility))))
            step_x, step_y = bx[i][1] == hi, by[j][1] == hi
            i, j, lo = i + step_x, j + step_y, hi
        if i < len(bx) or j < len(by):
            raise StrideConflict("the two factorisations do not cover the same extent")
        merged.append(dim)
    out = LayoutConstraint(c1.dims, merged)
    _check_chain(out)
    return out


def build_constraint(f, vector_elems, dims):
    """The constraint one copy puts on the buffer layout: each thread's ``vector_elems`` consecutive
    values must sit at consecutive addresses; every other stride stays free. LayoutIncompatible when
    the access is not a bijection onto the buffer."""
    f = filter_replication(f)
    total = math.prod(dims)
    if f.threads * f.values != total:
        raise LayoutIncompatible(f"the access covers {f.threads * f.values} of {total} elements")
    try:
        runs = inverse(f.layout).runs
    except NotInvertible as e:
        raise LayoutIncompatible(str(e)) from e
    T = f.threads
    vec_cuts = (T, T * vector_elems)
    dim_ends = list(np.cumprod(dims, dtype=object))
    splits = [[] for _ in dims]
    logical = 1
    for extent, tv_weight in runs:
        points = sorted(set(_refine(extent, tv_weight, vec_cuts)) | set(_refine(extent, logical, dim_ends)))
        prev = 1
        for p in points + [extent]:
            if p % prev or extent % p:
                raise LayoutIncompatible(f"cannot cut a run of {extent} at {p}")
            n = p // prev
            if n > 1 or (prev == 1 and p == extent):
                w, lw = tv_weight * prev, logical * prev
                dim = next(i for i, end in enumerate(dim_ends) if lw < end)
                entry = w // T if T <= w < T * vector_elems else StrideVar(vector_elems)
                _append_merging(splits[dim], n, entry)
            prev = p
        logical *= extent
    return LayoutConstraint(tuple(dims), [dim or [(1, StrideVar(1))] for dim in splits])


def parse_constraint(text):
    """``"((8,8),64):((1,D1),D2)"`` -> constraint; equal variable names are one variable."""
    body = "".join(text.split())
    try:
        shape_txt, stride_txt = body.split(":")
    except ValueError:
        raise LayoutIncompatible(f"constraint text {text!r} needs one ':'") from None
    shape_items, stride_items = _items(shape_txt), _items(stride_txt)
    if len(shape_items) != len(stride_items):
        raise LayoutIncompatible("constraint shape and stride have different dimension counts")
    free = {}
    splits = []
    for sh, st in zip(shape_items, stride_items):
        if isinstance(sh, list) is not isinstance(st, list):
            raise LayoutIncompatible("constraint dimension nests differently in shape and stride")
        sh, st = (sh, st) if isinstance(sh, list) else ([sh], [st])
        splits.append([(int(e), int(s) if s.isdigit() else free.setdefault(s, StrideVar())) for e, s in zip(sh, st)])
    return LayoutConstraint(tuple(math.prod(e for e, _ in dim) for dim in splits), splits)


def check_tma(c, element_bits, *, max_dims=5, align_bytes=16, max_box=256):
    """Can a bulk tensor copy serve this buffer? Few enough pieces, every extent within the box cap,
    a 16-byte contiguous innermost run; the hint materialises the free strides."""
    pieces, run_bytes = sum(map(len, c.splits)), _contiguous_run(c) * element_bits // 8
    for broken, reason in ((pieces > max_dims, f"{pieces} dims exceed limit {max_dims}"),
                           (max(c.dims) > max_box, f"extent exceeds box cap {max_box}"),
                           (run_bytes < align_bytes, f"innermost contiguous run is {run_bytes}B < {align_bytes}B")):
        if broken:
            return TmaCheck(False, reason)
    try:
        hint = materialize(c)
    except Unsatisfiable as e:
        return TmaCheck(False, str(e))
    return TmaCheck(True, "", hint)


def score_swizzles(generators, candidates=()):
    """Candidate with the least summed conflict degree over every generator's patterns (identity is
    always a candidate; ineligible swizzles -- ones that split a vector -- are skipped)."""
    pool = list(candidates) or candidate_swizzles()
    if IDENTITY_SWIZZLE not in pool:
        pool.insert(0, IDENTITY_SWIZZLE)
    totals = []
    for sw in pool:
        try:
            totals.append((sum(bank_conflicts(p, sw) for gen in generators for p in gen(sw)), sw))
        except MisalignedAccess:
            continue
    return _choose(totals)


def score_pattern_matrix(groups, pool):
    """Batched scoring: ``groups`` holds (patterns [P, lanes] of pre-swizzle byte addresses, width)
    per access width. Every swizzle of ``pool`` is applied to every pattern in one array
    expression. Returns (best swizzle, its total, per-swizzle totals with -1 for ineligible)."""
    sws = np.asarray([tuple(s) for s in pool], dtype=np.int64).reshape(-1, 3)
    bits, base, shift = (sws[:, i][:, None, None] for i in range(3))
    mask = (np.int64(1) << bits) - 1
    totals = np.zeros(len(pool), dtype=np.int64)
    eligible = np.ones(len(pool), dtype=bool)
    for pats, width in groups:
        a = pats[None].astype(np.int64)
        swz = a ^ (((a >> (base + shift)) & mask) << base)
        eligible &= ~((swz % width) != 0).any(axis=(1, 2))
        totals += phase_degrees(swz, width).sum(axis=-1)
    ranked = [(int(t), sw) for t, sw, ok in zip(totals, pool, eligible) if ok]
    best, total = _choose(ranked)
    return best, total, np.where(eligible, totals, -1)


def bank_conflicts(pattern, swizzle=IDENTITY_SWIZZLE):
    """Worst-phase conflict degree of one pattern (1 = conflict-free, also for no addresses)."""
    addrs = swizzle(np.asarray(pattern.addresses, dtype=np.int64))
    if addrs.size and (addrs % pattern.width).any():
        raise MisalignedAccess(f"{swizzle} breaks {pattern.width}-byte alignment")
    return int(phase_degrees(addrs, pattern.width))


def phase_degrees(addrs, width):
    """Conflict degree of every pattern: ``addrs`` is [..., lanes] of (already swizzled, aligned)
    byte addresses; returns [...] = max over phases and banks of the distinct words per bank
    (at least 1)."""
    lanes = addrs.shape[-1]
    if lanes == 0:
        return np.ones(addrs.shape[:-1], dtype=np.int64)
    words_each = max(1, width // BANK_BYTES)
    per_phase = lanes if width <= BANK_BYTES else max(1, lanes * BANK_BYTES // width)
    n_phase = -(-lanes // per_phase)
    pad = n_phase * per_phase - lanes
    if pad:  # a short last phase: repeat its first lane (a duplicate word changes no count)
        filler = np.repeat(addrs[..., (n_phase - 1) * per_phase:(n_phase - 1) * per_phase + 1], pad, axis=-1)
        addrs = np.concatenate([addrs, filler], axis=-1)
    words = addrs // BANK_BYTES
    if words_each > 1:
        words = (words[..., None] + np.arange(words_each)).reshape(*words.shape[:-1], -1)
    words = words.reshape(*addrs.shape[:-1], n_phase, per_phase * words_each)
    # sort each phase's words by (bank, word): equal words are neighbours, banks are runs
    key = np.sort((words % NUM_BANKS) << 40 | words, axis=-1)
    fresh = np.ones(key.shape, dtype=bool)
    fresh[..., 1:] = key[..., 1:] != key[..., :-1]
    bank = key >> 40
    starts = np.ones(key.shape, dtype=bool)
    starts[..., 1:] = bank[..., 1:] != bank[..., :-1]
    distinct = np.cumsum(fresh, axis=-1)
    before = np.maximum.accumulate(np.where(starts, distinct - fresh, 0), axis=-1)
    degree = (distinct - before).max(axis=(-1, -2))
    return np.maximum(degree, 1)


def _contiguous_run(c):
    run = 1
    for e, s in sorted(c.concrete_modes(), key=lambda m: m[1]):
        run *= e if s == run else 1
    return run


def _check_chain(c):
    """Concrete pieces, by stride, must stack into a bijection's stride chain."""
    reach = 1
    for e, s in sorted(c.concrete_modes(), key=lambda m: m[1]):
        if s < reach or s % reach:
            raise StrideConflict(f"concrete piece {e}:{s} overlaps the span {reach} below it")
        reach = s * e


def _sub_entry(piece, lo):
    start, _, s = piece
    return s * (lo // start) if isinstance(s, int) else StrideVar(s.divisibility)


# ------------------------------------------------------------------------------------------- unify
def _bounds(pieces):
    """(start, end, entry) of each piece on the cumulative-extent axis."""
    out, at = [], 1
    for e, s in pieces:
        out.append((at, at * e, s))
        at *= e
    return out


def _append_merging(dim, n, entry):
    """Append a piece; two neighbouring free pieces of one dimension become one free piece."""
    if dim and isinstance(entry, StrideVar) and isinstance(dim[-1][1], StrideVar):
        m, other = dim[-1]
        dim[-1] = (m * n, StrideVar(max(other.divisibility, entry.divisibility)))
    else:
        dim.append((n, entry))


# ------------------------------------------------------------------------------------------- build
def _refine(extent, weight, cuts):
    """Local cut points (1 < p < extent) of a run covering weights [weight, weight * extent) at the
    given global boundaries; a boundary inside the run must be a multiple of ``weight``."""
    out = []
    for b in cuts:
        if weight < b < weight * extent:
            if b % weight:
                raise LayoutIncompatible(f"boundary {b} is not aligned to the run weight {weight}")
            out.append(b // weight)
    return out


def _items(text):
    if not (text.startswith("(") and text.endswith(")")):
        raise LayoutIncompatible(f"constraint part {text!r} is not parenthesised")
    return [g.split(",") if g is not None else w for g, w in ((m.group(1), m.group(2))
                                                            for m in _ITEM.finditer(text[1:-1]))]


def _choose(totals):
    if not totals:
        return IDENTITY_SWIZZLE, 0
    total, sw = min(totals, key=lambda ts: (ts[0], tuple(ts[1])))
    return sw, total


def candidate_swizzles(min_base=2):
    """Identity plus the 1..3-bit XOR swizzles with target base 2..4 (>= ``min_base``, so vector
    atoms of 2^min_base bytes stay whole) and source shift up to 6."""
    return [IDENTITY_SWIZZLE] + [Swizzle(bits, base, shift) for bits in (1, 2, 3) for base in (2, 3, 4)
                                 if base >= min_base for shift in range(bits, 7)]


def apply_swizzle(s, addr):
    return s(addr)
