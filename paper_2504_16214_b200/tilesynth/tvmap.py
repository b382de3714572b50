"""Thread-value layouts: two-mode layouts (thread, value) -> position in a tile.

Contract: /root/reference/pkg/src/tilesynth/tv.py:1-156 (TvLayout, tv_from_mode_lists, restrict_tv,
filter_replication, tv_coalesced_key). Here a TvLayout is a value object over a :class:`Layout`
that can materialise its whole (threads x values) position grid as a numpy array; bijectivity,
surjectivity and pointwise equality are array comparisons on that grid, and the shared-memory
passes read the grid directly instead of evaluating positions one at a time.
"""
from __future__ import annotations

import math
from typing import Tuple

import numpy as np

from . import ituple
from .algebra import Layout, coalesce, restrict_mode_split
from .errors import NonBijectiveLayout, ShapeMismatch

Run = Tuple[int, int]


class TvLayout:
    """``layout`` has exactly two top-level modes (thread, value); ``tile`` gives the extents used
    to decode a position back into coordinates (first extent fastest)."""

    __slots__ = ("layout", "tile", "_t_runs", "_v_runs", "_grid")

    def __init__(self, layout, tile):
        if layout.rank != 2:
            raise ShapeMismatch(f"a thread-value layout has two modes, {layout} has {layout.rank}")
        object.__setattr__(self, "layout", layout)
        object.__setattr__(self, "tile", tuple(tile))
        object.__setattr__(self, "_t_runs", tuple(zip(ituple.leaves(layout.shape[0]), ituple.leaves(layout.stride[0]))))
        object.__setattr__(self, "_v_runs", tuple(zip(ituple.leaves(layout.shape[1]), ituple.leaves(layout.stride[1]))))
        object.__setattr__(self, "_grid", None)

    def __setattr__(self, name, value):
        raise AttributeError("TvLayout is immutable")

    def __eq__(self, other):
        return type(other) is TvLayout and (self.layout, self.tile) == (other.layout, other.tile)

    def __hash__(self):
        return hash((self.layout, self.tile))

    def __repr__(self):
        return f"TvLayout(layout={self.layout!r}, tile={self.tile!r})"

    def __str__(self):
        return str(self.layout)

    @property
    def threads(self):
        return math.prod(e for e, _ in self._t_runs)

    @property
    def values(self):
        return math.prod(e for e, _ in self._v_runs)

    @property
    def tile_size(self):
        return math.prod(self.tile)

    def grid(self):
        """positions[t, v] for the whole domain (int64, read-only, built once)."""
        if self._grid is None:
            def axis(runs):
                acc = np.zeros(1, dtype=np.int64)
                for e, d in runs:
                    acc = np.add.outer(np.arange(e, dtype=np.int64) * d, acc).ravel()
                return acc
            g = np.add.outer(axis(self._t_runs), axis(self._v_runs))
            g.flags.writeable = False
            object.__setattr__(self, "_grid", g)
        return self._grid

    def position(self, t, v):
        if not (0 <= t < self.threads and 0 <= v < self.values):
            raise ShapeMismatch(f"(thread {t}, value {v}) is outside {self.threads} x {self.values}")
        pos = 0
        for runs, x in ((self._t_runs, t), (self._v_runs, v)):
            for e, d in runs:
                x, r = divmod(x, e)
                pos += r * d
        return pos

    def coords(self, t, v):
        return ituple.decode(self.position(t, v), self.tile)

    def _covers_once(self):
        flat = np.sort(self.grid(), axis=None)
        return flat.size == self.tile_size and bool((flat == np.arange(flat.size)).all())

    def check_bijective(self, name="layout"):
        """Raise NonBijectiveLayout unless every tile position is hit exactly once."""
        if self.threads * self.values != self.tile_size:
            raise NonBijectiveLayout(f"{name}: {self.threads} x {self.values} values for a tile of "
                                     f"{self.tile_size}")
        if not self._covers_once():
            raise NonBijectiveLayout(f"{name} does not map onto its tile one-to-one")

    def is_surjective(self):
        hit = np.unique(self.grid())
        return hit.size == self.tile_size and bool((hit == np.arange(self.tile_size)).all())

    def same_function(self, other):
        """Pointwise equality over the (thread, value) domain (tiles of equal size)."""
        if (self.threads, self.values, self.tile_size) != (other.threads, other.values, other.tile_size):
            return False
        return tv_coalesced_key(self) == tv_coalesced_key(other) or bool((self.grid() == other.grid()).all())


def make_tv(layout, tile):
    return TvLayout(layout, tile)


def _pack(runs):
    kept = [r for r in runs if r[0] > 1]
    if not kept:
        return 1, 0
    if len(kept) == 1:
        return kept[0]
    return tuple(e for e, _ in kept), tuple(d for _, d in kept)


def tv_from_mode_lists(thread_modes, value_modes, tile):
    """TV layout from flat (extent, stride) runs per mode; unit runs are dropped."""
    (ts, td), (vs, vd) = _pack(thread_modes), _pack(value_modes)
    return TvLayout(Layout((ts, vs), (td, vd)), tile)


def restrict_tv(tv, threads, values):
    """The colex-fastest (threads x values) sub-domain, plus the dropped thread / value runs (the
    outer repetition digits)."""
    inner, spare_t = restrict_mode_split(tv.layout, 0, threads)
    inner, spare_v = restrict_mode_split(inner, 1, values)
    return TvLayout(inner, tv.tile), spare_t, spare_v


def filter_replication(tv):
    """Drop broadcast (stride-0) digits: the de-duplicated access sub-layout."""
    return tv_from_mode_lists([r for r in tv._t_runs if r[1]], [r for r in tv._v_runs if r[1]], tv.tile)


def tv_coalesced_key(tv):
    """Canonical key: coalesced thread and value modes plus the tile."""
    t, v = coalesce(tv.layout.mode(0)), coalesce(tv.layout.mode(1))
    return t.shape, t.stride, v.shape, v.stride, tv.tile
