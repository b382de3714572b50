"""Instruction catalogs: data-driven models of the collective copy / matrix / ALU instructions the
synthesizer may choose, loaded from ``data/<arch>.cat``.

Contract: /root/reference/pkg/src/tilesynth/catalog.py:1-338 -- the record format (``copy`` /
``mma`` / ``alu`` records of ``key value`` lines closed by ``end``, header keys, the ``generic``
and ``tma`` flags), the validation rules, and the queries ``candidates_for_copy`` (widest vector
first), ``tma_candidates`` and ``fastest_mma`` (best issue cycles per MAC).

Construction here: the file is split into records by a small generator; each record kind has a
schema (allowed keys, required keys) and a builder; explicit thread-value layouts are checked for
bijectivity through :class:`algebra.TvLayout`'s grid.
"""
from __future__ import annotations

import math
from dataclasses import field, make_dataclass
from pathlib import Path

from .algebra import Layout, parse_layout
from .errors import CatalogFormatError, NoInstructionAvailable
from .algebra import TvLayout

DATA_DIR = Path(__file__).resolve().parent / "data"


class _InstructionOps:
    """Behaviour of a catalog entry (the fields are declared in ``_FIELDS`` below)."""

    __slots__ = ()

    def vector_elems(self, dtype):
        return self.vector_bytes * 8 // (self.element_bits or dtype.bits)

    def supports_dtype(self, dtype):
        if self.category != "copy":
            return False
        if self.element_bits:
            return dtype.bits == self.element_bits
        return 8 * self.vector_bytes >= dtype.bits and (8 * self.vector_bytes) % dtype.bits == 0

    def copy_layouts(self, dtype):
        """(source, destination) thread-value layouts in element units. A generic entry moves
        ``vector_bytes`` of consecutive elements per thread; its modes are one-element tuples so
        that composition keeps the (thread, value) structure."""
        if self.category != "copy" or self.tma:
            raise NoInstructionAvailable(f"{self.name} has no thread-value layouts")
        if not self.generic:
            return tuple(TvLayout(lay, self.tile) for lay in (self.tv_src, self.tv_dst))
        v = self.vector_elems(dtype)
        lanes = ((self.threads,), (v,)) if v > 1 else ((self.threads,), (1,))
        steps = ((v,), (1,)) if v > 1 else ((1,), (0,))
        one = TvLayout(Layout(lanes, steps), (self.threads * v,))
        return one, one

    def mma_layouts(self):
        m, n, k = self.mnk
        return tuple(TvLayout(lay, ext) for lay, ext in ((self.tv_a, (m, k)), (self.tv_b, (n, k)), (self.tv_c, (m, n))))

    def macs(self):
        return math.prod(self.mnk)


# (field, default) after the four required ones (name, category, issue_cycles, completion_cycles)
_FIELDS = (
    ("arch", ""),
    # copies: scopes, vector width, thread count, generic / TMA flags, explicit per-tile layouts
    ("src_scope", None), ("dst_scope", None), ("vector_bytes", 0), ("threads", 0), ("generic", False),
    ("element_bits", 0), ("tile", ()), ("tv_src", None), ("tv_dst", None), ("tma", False),
    # matrix instructions: shape, operand dtypes, fragment layouts
    ("mnk", ()), ("dtype_a", None), ("dtype_b", None), ("dtype_c", None), ("tv_a", None), ("tv_b", None),
    ("tv_c", None),
)
Instruction = make_dataclass(
    "Instruction", ["name", "category", "issue_cycles", "completion_cycles"]
    + [(f, object, field(default=d)) for f, d in _FIELDS], bases=(_InstructionOps,), frozen=True,
    namespace={"__module__": __name__})


class Catalog:
    """An architecture's instructions plus its memory-system parameters."""

    _PARAMS = (("banks", 32), ("bank_bytes", 4), ("tma_max_dims", 5), ("tma_align_bytes", 16), ("tma_max_box", 256))

    def __init__(self, arch, instructions, **params):
        unknown = set(params) - {p for p, _ in self._PARAMS}
        if unknown:
            raise TypeError(f"unknown catalog parameters {sorted(unknown)}")
        self.arch, self.instructions = arch, list(instructions)
        for p, default in self._PARAMS:
            setattr(self, p, params.get(p, default))
        self.by_name = {i.name: i for i in self.instructions}

    def alu(self):
        return next((i for i in self.instructions if i.category == "alu"),
                    Instruction("alu_default", "alu", 1, 8, self.arch))


# --------------------------------------------------------------------------------------- the format
_HEADER = ("banks", "bank_bytes", "tma_max_dims", "tma_align_bytes", "tma_max_box")
_FLAGS = ("generic", "tma")
_SCHEMA = {  # kind -> allowed keys
    "copy": {"scopes", "vector_bytes", "threads", "issue", "completion", "generic", "element_bits", "tile",
             "tv_src", "tv_dst", "tma"},
    "mma": {"mnk", "dtypes", "tv_a", "tv_b", "tv_c", "threads", "issue", "completion"},
    "alu": {"issue", "completion"},
}
_SCOPE_NAMES = {"Global", "Shared", "Register"}


def _records(text, header):
    """Yield (kind, name, fields) per record; header lines fill ``header``."""
    open_rec = None
    for lineno, raw in enumerate(text.splitlines(), start=1):
        words = raw.split("#", 1)[0].split(None, 1)
        if not words:
            continue
        key, value = words[0], (words[1].strip() if len(words) > 1 else "")
        if open_rec is not None:
            if key == "end":
                yield open_rec
                open_rec = None
            else:
                open_rec[2][key] = "true" if key in _FLAGS and not value else value
        elif key == "catalog":
            if "arch" in header:
                raise CatalogFormatError(f"line {lineno}: duplicate catalog header")
            header["arch"] = value
        elif key in _HEADER:
            header[key] = int(value)
        elif key in _SCHEMA:
            if not value:
                raise CatalogFormatError(f"line {lineno}: record needs a name")
            open_rec = (key, value, {})
        else:
            raise CatalogFormatError(f"line {lineno}: unknown key {key!r}")
    if open_rec is not None:
        raise CatalogFormatError("unterminated instruction record")


def _tile(text):
    body = text.strip()
    if body[:1] != "(" or body[-1:] != ")":
        raise CatalogFormatError(f"bad tile {text!r}")
    return tuple(map(int, body[1:-1].split(",")))


class _Record:
    """One catalog record being turned into an :class:`Instruction`; every complaint names it."""

    def __init__(self, kind, name, fields, arch):
        self.kind, self.name, self.fields, self.arch = kind, name, fields, arch

    def reject(self, why):
        raise CatalogFormatError(f"instruction {self.name}: {why}")

    def need(self, key):
        return self.fields[key] if key in self.fields else self.reject(f"missing key {key!r}")

    def ensure(self, ok, why):
        if not ok:
            self.reject(why)

    def build(self):
        issue, completion = int(self.need("issue")), int(self.need("completion"))
        self.ensure(min(issue, completion) >= 1, "cycles must be >= 1")
        stray = sorted(set(self.fields) - _SCHEMA[self.kind])
        self.ensure(not stray, f"unknown keys {stray}")
        spec = dict(name=self.name, category=self.kind, issue_cycles=issue, completion_cycles=completion,
                    arch=self.arch)
        if self.kind != "alu":
            spec["threads"] = int(self.fields.get("threads", "32"))
        inst = Instruction(**spec, **getattr(self, "_" + self.kind)())
        for label, tv in self._explicit_layouts(inst):
            tv.check_bijective(f"{self.name}.{label}")
            self.ensure(self.kind == "mma" or tv.threads == inst.threads, "thread mode size != threads field")
        return inst

    def _alu(self):
        return {}

    def _mma(self):
        shape, types = tuple(map(int, self.need("mnk").split())), self.need("dtypes").split()
        self.ensure(len(shape) == 3 and len(types) == 3, "mnk and dtypes take three values each")
        out = dict(mnk=shape, dtype_a=types[0], dtype_b=types[1], dtype_c=types[2])
        out.update((k, parse_layout(self.need(k))) for k in ("tv_a", "tv_b", "tv_c"))
        return out

    def _copy(self):
        scopes = self.need("scopes").split()
        self.ensure(len(scopes) == 2 and set(scopes) <= _SCOPE_NAMES, f"bad scopes {scopes}")
        width = int(self.need("vector_bytes"))
        self.ensure(width in (1, 2, 4, 8, 16), "vector_bytes must be one of 1,2,4,8,16")
        out = dict(src_scope=scopes[0], dst_scope=scopes[1], vector_bytes=width, generic="generic" in self.fields,
                   tma="tma" in self.fields, element_bits=int(self.fields.get("element_bits", "0")))
        convert = {"tile": _tile, "tv_src": parse_layout, "tv_dst": parse_layout}
        out.update((k, conv(self.fields[k])) for k, conv in convert.items() if k in self.fields)
        return out

    def _explicit_layouts(self, inst):
        if self.kind == "mma":
            return zip(("tv_a", "tv_b", "tv_c"), inst.mma_layouts())
        if self.kind == "alu" or inst.generic or inst.tma:
            return ()
        self.ensure(inst.tv_src is not None and inst.tv_dst is not None and inst.tile,
                    "explicit entries need tile, tv_src, tv_dst")
        return zip(("tv_src", "tv_dst"), inst.copy_layouts(None))


def load_catalog(path):
    """Load and validate a catalog file (unknown keys rejected, explicit layouts must be bijections
    onto their tiles, names unique)."""
    header = {}
    insts = [_Record(kind, name, fields, str(header.get("arch") or "")).build()
             for kind, name, fields in _records(Path(path).read_text(), header)]
    if "arch" not in header or not insts:
        raise CatalogFormatError("catalog needs a header and at least one instruction")
    if len({i.name for i in insts}) != len(insts):
        raise CatalogFormatError("duplicate instruction names")
    arch = header.pop("arch")
    return Catalog(arch, insts, **header)


def builtin_catalog_path(arch="sm80"):
    return DATA_DIR / f"{arch}.cat"


# ------------------------------------------------------------------------------------------ queries
def _pick(cat, category, **want):
    """Catalog entries of ``category`` whose attributes equal ``want`` (in catalog order)."""
    return [i for i in cat.instructions
            if i.category == category and all(getattr(i, k) == v for k, v in want.items())]


def candidates_for_copy(cat, src, dst):
    """Instructions able to move ``src`` -> ``dst`` (widest vector first, then by name; the last is
    the scalar fallback). A register-to-register move needs none: []."""
    if src.scope == dst.scope == "Register":
        return []
    fits = [i for i in _pick(cat, "copy", tma=False, src_scope=src.scope, dst_scope=dst.scope)
            if i.supports_dtype(src.dtype)]
    if not fits:
        raise NoInstructionAvailable(f"no copy instruction for {src.scope}->{dst.scope} {src.dtype}")
    return sorted(fits, key=lambda i: (-i.vector_bytes, i.name))


def tma_candidates(cat, src, dst):
    return _pick(cat, "copy", tma=True, src_scope=src.scope, dst_scope=dst.scope)


def fastest_mma(cat, a_dtype, b_dtype, c_dtype):
    """The matching matrix instruction with the fewest issue cycles per MAC (then by name)."""
    fits = _pick(cat, "mma", dtype_a=a_dtype.name, dtype_b=b_dtype.name, dtype_c=c_dtype.name)
    if not fits:
        raise NoInstructionAvailable(f"no matrix instruction for {a_dtype} x {b_dtype} -> {c_dtype}")
    return min(fits, key=lambda i: (i.issue_cycles / i.macs(), i.name))
