"""XOR swizzles over byte addresses and a vectorised shared-memory bank-conflict model.

Contract: /root/reference/pkg/src/tilesynth/swizzle.py:1-160 -- the swizzle family, the bank model
(32 banks x 4 B; an 8-byte access runs in 2 phases of 16 threads, a 16-byte access in 4 phases of
8; the degree of a phase is the largest number of distinct words one bank serves) and the scoring
rule (least total over the patterns, ties toward smaller (bits, base, shift), swizzles that would
split a vector are ineligible).

The model is evaluated on whole arrays: a batch of warp-wide access patterns (rows of an int64
matrix) against every candidate swizzle at once, so a buffer's swizzle search is one numpy pass
(:func:`score_pattern_matrix`) instead of a Python loop per (swizzle, pattern, lane).
"""
from __future__ import annotations

from typing import Callable, Iterable

import numpy as np

from .errors import MisalignedAccess

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


def apply_swizzle(s, addr):
    return s(addr)


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


def bank_conflicts(pattern, swizzle=IDENTITY_SWIZZLE):
    """Worst-phase conflict degree of one pattern (1 = conflict-free, also for no addresses)."""
    addrs = swizzle(np.asarray(pattern.addresses, dtype=np.int64))
    if addrs.size and (addrs % pattern.width).any():
        raise MisalignedAccess(f"{swizzle} breaks {pattern.width}-byte alignment")
    return int(phase_degrees(addrs, pattern.width))


PatternGenerator = Callable[[Swizzle], Iterable[AccessPattern]]


def candidate_swizzles(min_base=2):
    """Identity plus the 1..3-bit XOR swizzles with target base 2..4 (>= ``min_base``, so vector
    atoms of 2^min_base bytes stay whole) and source shift up to 6."""
    return [IDENTITY_SWIZZLE] + [Swizzle(bits, base, shift) for bits in (1, 2, 3) for base in (2, 3, 4)
                                 if base >= min_base for shift in range(bits, 7)]


def _choose(totals):
    if not totals:
        return IDENTITY_SWIZZLE, 0
    total, sw = min(totals, key=lambda ts: (ts[0], tuple(ts[1])))
    return sw, total


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
