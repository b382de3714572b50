"""Thread-value (TV) layouts: a two-mode layout (thread, value) -> linear position in a tile.

Semantics follow the reference (``/root/reference/pkg/src/tilesynth/tv.py:13-156``). Here a TV layout
also carries its whole image as a ``[threads, values]`` numpy grid (built once from the two modes'
tables), so bijectivity checks, pointwise comparisons and the shared-memory access patterns are
array operations instead of per-(thread, value) evaluation.
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

import numpy as np

from . import nested
from .errors import NonBijectiveLayout, ShapeMismatch
from .layout_algebra import Layout, coalesce, restrict_mode_split

Run = Tuple[int, int]


class TvLayout:
    """``layout`` has exactly two top-level modes (thread, value); ``tile`` decodes positions
    (first extent fastest)."""

    __slots__ = ("layout", "tile", "_t", "_v", "_grid")

    def __init__(self, layout: Layout, tile: Sequence[int]):
        if layout.rank != 2:
            raise ShapeMismatch(f"thread-value layout needs exactly 2 modes, got {layout}")
        tm, vm = layout.mode(0), layout.mode(1)
        for name, value in (("layout", layout), ("tile", tuple(tile)), ("_t", tm), ("_v", vm), ("_grid", None)):
            object.__setattr__(self, name, value)

    def __setattr__(self, name, value):
        raise AttributeError("TvLayout is frozen")

    def __eq__(self, other) -> bool:
        return isinstance(other, TvLayout) and self.layout == other.layout and self.tile == other.tile

    def __hash__(self) -> int:
        return hash((self.layout, self.tile))

    def __repr__(self) -> str:
        return f"TvLayout(layout={self.layout!r}, tile={self.tile!r})"

    def __str__(self) -> str:
        return str(self.layout)

    # ------------------------------------------------------------------------------------------
    @property
    def threads(self) -> int:
        return self._t.size()

    @property
    def values(self) -> int:
        return self._v.size()

    @property
    def tile_size(self) -> int:
        return nested.size(self.tile) if self.tile else 1

    def position(self, t: int, v: int) -> int:
        if not (0 <= t < self._t.size() and 0 <= v < self._v.size()):
            raise ShapeMismatch(f"(t={t}, v={v}) outside layout domain")
        return self._t(t) + self._v(v)

    def coords(self, t: int, v: int) -> Tuple[int, ...]:
        return nested.decode(self.position(t, v), self.tile)

    def grid(self) -> np.ndarray:
        """positions[t, v] for the whole domain (int64, cached, read-only)."""
        if self._grid is None:
            g = self._t.table()[:, None] + self._v.table()[None, :]
            g.setflags(write=False)
            object.__setattr__(self, "_grid", g)
        return self._grid

    def check_bijective(self, name: str = "layout") -> None:
        n = self.tile_size
        if self.threads * self.values != n:
            raise NonBijectiveLayout(f"{name}: {self.threads}x{self.values} values vs tile of {n}")
        image = np.unique(self.grid())
        if image.size != n or image[0] != 0 or image[-1] != n - 1:
            raise NonBijectiveLayout(f"{name} is not a bijection onto its tile")

    def is_surjective(self) -> bool:
        image = np.unique(self.grid())
        n = self.tile_size
        return image.size == n and image[0] == 0 and image[-1] == n - 1

    def same_function(self, other: "TvLayout") -> bool:
        """Pointwise equality over the whole (thread, value) domain."""
        if (self.threads, self.values, self.tile_size) != (other.threads, other.values, other.tile_size):
            return False
        return tv_coalesced_key(self) == tv_coalesced_key(other) or bool(np.array_equal(self.grid(), other.grid()))


def make_tv(layout: Layout, tile: Sequence[int]) -> TvLayout:
    return TvLayout(layout, tuple(tile))


def _one_mode(runs: Sequence[Run]):
    runs = [r for r in runs if r[0] > 1]
    if not runs:
        return 1, 0
    if len(runs) == 1:
        return runs[0]
    return tuple(e for e, _ in runs), tuple(d for _, d in runs)


def tv_from_mode_lists(thread_modes: Sequence[Run], value_modes: Sequence[Run], tile: Sequence[int]) -> TvLayout:
    """Assemble (thread runs, value runs) into a TV layout; unit runs vanish and a single run
    becomes a scalar mode."""
    (ts, td), (vs, vd) = _one_mode(thread_modes), _one_mode(value_modes)
    return TvLayout(Layout((ts, vs), (td, vd)), tuple(tile))


def restrict_tv(tv: TvLayout, threads: int, values: int) -> Tuple[TvLayout, List[Run], List[Run]]:
    """The colex-fastest (threads x values) sub-domain, plus the dropped thread and value runs."""
    inner, drop_t = restrict_mode_split(tv.layout, 0, threads)
    inner, drop_v = restrict_mode_split(inner, 1, values)
    return TvLayout(inner, tv.tile), drop_t, drop_v


def filter_replication(tv: TvLayout) -> TvLayout:
    """Drop broadcast (stride-0) digits of both modes."""
    keep = lambda m: [(e, d) for e, d in m.flat_modes() if d and e > 1]  # noqa: E731
    return tv_from_mode_lists(keep(tv._t), keep(tv._v), tv.tile)


def tv_coalesced_key(tv: TvLayout) -> Tuple:
    t, v = coalesce(tv._t), coalesce(tv._v)
    return t.shape, t.stride, v.shape, v.stride, tv.tile
