"""Error taxonomy of the layout synthesizer.

The class names and their is-a relations are the public contract -- callers (and the reference's
own tests, run against this package through ``compat/``) catch ``LayoutError`` or a specific leaf
such as ``NotInvertible`` -- so they follow /root/reference/pkg/src/tilesynth/errors.py:1-124.
The leaves are generated from one table; only the two errors that carry data are written out.
"""
from __future__ import annotations


class TileSynthError(Exception):
    """Root of everything the synthesizer raises."""


class ParseError(TileSynthError):
    """Malformed program, layout or tuple text; ``line`` / ``column`` locate it when known."""

    def __init__(self, message, line=0, column=0):
        self.line, self.column = line, column
        super().__init__(f"line {line}, col {column}: {message}" if line else message)


class ConflictDetected(TileSynthError):
    """One tensor was handed two different thread-value layouts."""

    def __init__(self, tensor, existing, incoming, op_index):
        self.tensor, self.existing, self.incoming, self.op_index = tensor, existing, incoming, op_index
        super().__init__(f"op {op_index} assigns tensor '{tensor}' the layout {incoming}, "
                         f"but it already has {existing}")


# (class, parent, what it means)
_TAXONOMY = (
    ("LayoutError", "TileSynthError", "Layout-algebra failure."),
    ("ShapeMismatch", "LayoutError", "A coordinate or operand does not fit the shape tree."),
    ("OutOfDomain", "LayoutError", "An index or coordinate lies outside a layout's domain."),
    ("LayoutIncompatible", "LayoutError", "Two layouts cannot be combined (divisibility)."),
    ("NotInvertible", "LayoutError", "Not a bijection onto a contiguous index range."),
    ("NotComplementable", "LayoutError", "No gap-filling layout for the requested codomain."),
    ("NotDivisible", "LayoutError", "A mode cannot be cut at the requested extent."),
    ("IntegerOverflow", "LayoutError", "An extent, stride or index leaves the 64-bit range."),
    ("MisalignedAccess", "TileSynthError", "A vector access is not aligned to its width."),
    ("UnknownTensor", "TileSynthError", "A statement names a tensor that was never declared."),
    ("ArityError", "TileSynthError", "An operation got the wrong operand roles."),
    ("UnknownOp", "TileSynthError", "An operation index is out of range."),
    ("CatalogFormatError", "TileSynthError", "Malformed instruction catalog."),
    ("NonBijectiveLayout", "TileSynthError", "A catalog layout does not cover its tile exactly once."),
    ("NoInstructionAvailable", "TileSynthError", "No catalog instruction fits the request."),
    ("NonDivisibleTile", "TileSynthError", "A tensor extent does not divide by the tiling."),
    ("UnsolvedResidual", "TileSynthError", "Constraints left after propagation reached a fixpoint."),
    ("StrideConflict", "TileSynthError", "Buffer constraints force two elements onto one address."),
    ("Unsatisfiable", "TileSynthError", "Stride variables admit no bijective assignment."),
)

for _cls, _base, _doc in _TAXONOMY:
    globals()[_cls] = type(_cls, (globals()[_base],), {"__doc__": _doc, "__module__": __name__})


__all__ = ["TileSynthError", "ParseError", "ConflictDetected"] + [row[0] for row in _TAXONOMY]
