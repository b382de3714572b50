"""XOR swizzles and the shared-memory bank model, vectorised with numpy.

Bank model (the reference's, ``/root/reference/pkg/src/tilesynth/swizzle.py:17-160``): 32 banks of
4-byte words. A warp access of width <= 4 B is one phase over all lanes; an 8 B access runs as
phases of 16 lanes, a 16 B access as phases of 8 lanes, each lane touching width/4 consecutive
words. A phase's conflict degree is the largest number of DISTINCT words that map to one bank;
a pattern's degree is the worst phase (>= 1).

Here a set of patterns is an int64 matrix ``[patterns, lanes]`` of byte addresses, and the degree
of every (swizzle, pattern, phase) is computed at once: swizzle by broadcasting, expand lanes into
words, sort each phase, keep first occurrences, ``bincount`` (phase, bank) keys. The point-wise
API (:class:`AccessPattern`, :func:`bank_conflicts`, :func:`score_swizzles`) is kept on top of it.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Iterable, List, Sequence, Tuple

import numpy as np

from .errors import MisalignedAccess

NUM_BANKS = 32
BANK_BYTES = 4
VALID_WIDTHS = (1, 2, 4, 8, 16)


@dataclass(frozen=True, order=True)
class Swizzle:
    """``addr ^ (((addr >> (base + shift)) & (2^bits - 1)) << base)``; bits = 0 is the identity."""

    bits: int
    base: int
    shift: int

    def __post_init__(self):
        if min(self.bits, self.base) < 0:
            raise ValueError("swizzle fields must be nonnegative")
        if self.bits and self.shift < self.bits:
            raise ValueError("swizzle source and target fields overlap")

    def __call__(self, addr: int) -> int:
        if addr < 0:
            raise ValueError("swizzle expects a nonnegative address")
        return addr ^ (((addr >> (self.base + self.shift)) & ((1 << self.bits) - 1)) << self.base)

    def apply(self, addrs: np.ndarray) -> np.ndarray:
        """Vectorised :meth:`__call__` (addresses assumed nonnegative)."""
        if not self.bits:
            return addrs
        return addrs ^ (((addrs >> (self.base + self.shift)) & ((1 << self.bits) - 1)) << self.base)

    @property
    def is_identity(self) -> bool:
        return self.bits == 0

    def __str__(self) -> str:
        return f"SW({self.bits},{self.base},{self.shift})"


IDENTITY_SWIZZLE = Swizzle(0, 4, 3)


def apply_swizzle(s: Swizzle, addr: int) -> int:
    return s(addr)


def candidate_swizzles(min_base: int = 2) -> List[Swizzle]:
    """Identity plus SW(bits in 1..3, base in 2..4 with base >= min_base, shift in bits..6)."""
    family = [Swizzle(b, m, s) for b in (1, 2, 3) for m in (2, 3, 4) if m >= min_base for s in range(b, 7)]
    return [IDENTITY_SWIZZLE] + family


# ------------------------------------------------------------------------------- vector kernel
def phase_degrees(addrs: np.ndarray, width: int) -> np.ndarray:
    """Conflict degree of each pattern (row) of swizzled byte addresses ``[..., P, L]`` -> ``[..., P]``."""
    *lead, lanes = addrs.shape
    rows = int(np.prod(lead)) if lead else 1
    if lanes == 0:
        return np.ones(lead, dtype=np.int64)
    per_lane = max(1, width // BANK_BYTES) if width > BANK_BYTES else 1
    group = lanes if width <= BANK_BYTES else max(1, lanes * BANK_BYTES // width)
    n_phase = -(-lanes // group)
    a = addrs.reshape(rows, lanes)
    if n_phase * group != lanes:  # ragged last phase: pad with its own first lane (adds no new word)
        pad = np.repeat(a[:, (n_phase - 1) * group:(n_phase - 1) * group + 1], n_phase * group - lanes, axis=1)
        a = np.concatenate([a, pad], axis=1)
    words = a // BANK_BYTES
    if per_lane > 1:
        words = (words[:, :, None] + np.arange(per_lane)).reshape(rows, n_phase * group * per_lane)
    words = np.sort(words.reshape(rows * n_phase, group * per_lane), axis=1)
    fresh = np.ones(words.shape, dtype=bool)
    fresh[:, 1:] = words[:, 1:] != words[:, :-1]
    key = (np.arange(rows * n_phase)[:, None] * NUM_BANKS + words % NUM_BANKS)[fresh]
    per_bank = np.bincount(key, minlength=rows * n_phase * NUM_BANKS).reshape(rows * n_phase, NUM_BANKS)
    worst = per_bank.max(axis=1).reshape(rows, n_phase).max(axis=1)
    return np.maximum(worst, 1).reshape(lead) if lead else np.maximum(worst, 1)[0]


def score_pattern_sets(sets: Sequence[Tuple[np.ndarray, int]], pool: Sequence[Swizzle]):
    """For each swizzle of ``pool`` (already in scoring order): None when it breaks the alignment of
    any access of any set, else the per-set arrays of pattern degrees."""
    out = []
    for sw in pool:
        degrees = []
        for addrs, width in sets:
            moved = sw.apply(addrs)
            if width > 1 and (moved % width).any():
                degrees = None
                break
            degrees.append(phase_degrees(moved, width))
        out.append(degrees)
    return out


def best_swizzle(sets: Sequence[Tuple[np.ndarray, int]], pool: Sequence[Swizzle]) -> Tuple[Swizzle, int, list]:
    """The swizzle minimising the summed pattern degrees (ties -> smaller (bits, base, shift)); the
    identity always competes. Returns (swizzle, its total, its per-set degree arrays)."""
    pool = list(pool)
    if IDENTITY_SWIZZLE not in pool:
        pool.insert(0, IDENTITY_SWIZZLE)
    pool.sort(key=lambda s: (s.bits, s.base, s.shift))
    best = (None, IDENTITY_SWIZZLE, [])
    for sw, degrees in zip(pool, score_pattern_sets(sets, pool)):
        if degrees is None:
            continue
        key = (int(sum(int(d.sum()) for d in degrees)), sw.bits, sw.base, sw.shift)
        if best[0] is None or key < best[0]:
            best = (key, sw, degrees)
    return best[1], (best[0][0] if best[0] is not None else 0), best[2]


# ------------------------------------------------------------------------------- point-wise API
@dataclass(frozen=True)
class AccessPattern:
    """Byte addresses of one warp-wide access (one per lane) and its width."""

    addresses: Tuple[int, ...]
    width: int

    def __post_init__(self):
        if self.width not in VALID_WIDTHS:
            raise MisalignedAccess(f"unsupported access width {self.width}")
        bad = [a for a in self.addresses if a % self.width]
        if bad:
            raise MisalignedAccess(f"address {bad[0]} not aligned to width {self.width}")


def bank_conflicts(pattern: AccessPattern, swizzle: Swizzle = IDENTITY_SWIZZLE) -> int:
    """Worst-phase conflict degree of one pattern under ``swizzle`` (1 = conflict-free or empty)."""
    moved = [swizzle(a) for a in pattern.addresses]
    bad = [a for a in moved if a % pattern.width]
    if bad:
        raise MisalignedAccess(f"swizzled address {bad[0]} breaks {pattern.width}-byte alignment")
    return int(phase_degrees(np.asarray([moved], dtype=np.int64).reshape(1, len(moved)), pattern.width)[0])


PatternGenerator = Callable[[Swizzle], Iterable[AccessPattern]]


def score_swizzles(generators: Sequence[PatternGenerator], candidates: Sequence[Swizzle] = ()) -> Tuple[Swizzle, int]:
    """Pick the candidate minimising the total worst-phase degree over every generated pattern.
    A swizzle that misaligns any access is skipped; ties go to smaller (bits, base, shift), and the
    identity is always scored, so the result never loses to it."""
    pool = sorted(set(candidates or candidate_swizzles()) | {IDENTITY_SWIZZLE},
                  key=lambda s: (s.bits, s.base, s.shift))
    best_key, best_sw = None, IDENTITY_SWIZZLE
    for sw in pool:
        try:
            total = sum(bank_conflicts(p, sw) for gen in generators for p in gen(sw))
        except MisalignedAccess:
            continue
        if best_key is None or (total, sw.bits, sw.base, sw.shift) < best_key:
            best_key, best_sw = (total, sw.bits, sw.base, sw.shift), sw
    return best_sw, (best_key[0] if best_key else 0)
