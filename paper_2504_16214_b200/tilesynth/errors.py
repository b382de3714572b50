"""Exception types of the layout synthesizer.

The class NAMES and their subclass relations are the reference's public interface
(``/root/reference/pkg/src/tilesynth/errors.py:4-124``): callers catch them by name, and the
reference's own tests import them. They are declared here as one table -- (name, parent,
meaning) -- and materialised with ``type``; only the two classes that carry structured payloads
(:class:`ParseError`, :class:`ConflictDetected`) are written out.
"""
from __future__ import annotations

__all__: list[str] = []


class TileSynthError(Exception):
    """Root of every error raised by the synthesizer."""


# name -> (parent, one-line meaning). Order matters only in that parents precede children.
_TABLE = {
    # layout algebra
    "LayoutError": ("TileSynthError", "layout-algebra failure"),
    "ShapeMismatch": ("LayoutError", "coordinate / operand structure does not fit the shape"),
    "OutOfDomain": ("LayoutError", "index or coordinate outside a layout's domain"),
    "LayoutIncompatible": ("LayoutError", "operands violate a divisibility condition"),
    "NotInvertible": ("LayoutError", "not a bijection onto a contiguous range"),
    "NotComplementable": ("LayoutError", "no gap-filling layout for the codomain"),
    "NotDivisible": ("LayoutError", "a mode cannot be split at the requested size"),
    "IntegerOverflow": ("LayoutError", "value outside the supported 64-bit range"),
    # shared-memory banking
    "MisalignedAccess": ("TileSynthError", "an access is not aligned to its width"),
    # program IR
    "UnknownTensor": ("TileSynthError", "reference to an undeclared tensor"),
    "ArityError": ("TileSynthError", "wrong operand count / kind for an operation"),
    "UnknownOp": ("TileSynthError", "operation index out of range"),
    # instruction catalog
    "CatalogFormatError": ("TileSynthError", "malformed catalog text"),
    "NonBijectiveLayout": ("TileSynthError", "an instruction layout is not a bijection onto its tile"),
    "NoInstructionAvailable": ("TileSynthError", "no compatible instruction"),
    # synthesis
    "NonDivisibleTile": ("TileSynthError", "extent not divisible by the instruction / warp tiling"),
    "UnsolvedResidual": ("TileSynthError", "constraints left after propagation reached a fixpoint"),
    # shared memory
    "StrideConflict": ("TileSynthError", "unified constraints force duplicate addresses"),
    "Unsatisfiable": ("TileSynthError", "stride variables admit no bijective assignment"),
}

_ns = globals()
for _name, (_parent, _meaning) in _TABLE.items():
    _ns[_name] = type(_name, (_ns[_parent],), {"__doc__": _meaning[0].upper() + _meaning[1:] + ".",
                                               "__module__": __name__})


class ParseError(TileSynthError):
    """Malformed program / layout / catalog text; ``line`` and ``column`` locate it (0 = unknown)."""

    def __init__(self, message: str, line: int = 0, column: int = 0):
        self.line, self.column = line, column
        super().__init__(f"line {line}, col {column}: {message}" if line else message)


class ConflictDetected(TileSynthError):
    """Two different thread-value layouts demanded for one tensor (kept for API parity: synthesis
    resolves such conflicts with a redistribution instead of raising)."""

    def __init__(self, tensor: str, existing, incoming, op_index: int):
        self.tensor, self.existing, self.incoming, self.op_index = tensor, existing, incoming, op_index
        super().__init__(f"tensor '{tensor}' assigned two different thread-value layouts "
                         f"(op {op_index}): {existing} vs {incoming}")


__all__ += ["TileSynthError", "ParseError", "ConflictDetected", *_TABLE]
