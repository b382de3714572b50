"""Nested integer tuples ("IntTuples"): the shape / stride trees of layouts.

An IntTuple is an ``int`` or a ``tuple`` of IntTuples. Linear indices decompose
colexicographically: the leftmost leaf varies fastest. Semantics follow the reference's
``inttuple`` module (``/root/reference/pkg/src/tilesynth/inttuple.py:23-143``); the
implementation walks trees with explicit stacks and parses with a token state machine.
"""
from __future__ import annotations

import math
import re
from typing import Iterator, Tuple, Union

from .errors import IntegerOverflow, ParseError, ShapeMismatch

IntTuple = Union[int, Tuple["IntTuple", ...]]
INT64_MAX = (1 << 63) - 1


def is_int(t) -> bool:
    return isinstance(t, int)


def leaves(t: IntTuple) -> Iterator[int]:
    """Leaves left to right (colex order), without recursion."""
    stack = [t]
    while stack:
        node = stack.pop()
        if isinstance(node, tuple):
            stack.extend(reversed(node))
        else:
            yield node


def flatten(t: IntTuple) -> Tuple[int, ...]:
    return tuple(leaves(t))


def size(t: IntTuple) -> int:
    return math.prod(leaves(t))


def depth(t: IntTuple) -> int:
    best, stack = 0, [(t, 0)]
    while stack:
        node, d = stack.pop()
        if isinstance(node, tuple):
            best = max(best, d + 1)
            stack.extend((c, d + 1) for c in node)
    return best


def validate(t: IntTuple, *, min_leaf: int = 0) -> None:
    """Every leaf an int in [min_leaf, 2^63); anything else that is not a tuple is rejected."""
    stack = [t]
    while stack:
        node = stack.pop()
        if isinstance(node, tuple):
            stack.extend(reversed(node))
        elif not isinstance(node, int):
            raise ShapeMismatch(f"expected int or tuple, got {type(node).__name__}")
        elif node < min_leaf:
            raise ShapeMismatch(f"leaf {node} below minimum {min_leaf}")
        elif node > INT64_MAX:
            raise IntegerOverflow(f"leaf {node} exceeds 64-bit range")


def congruent(a: IntTuple, b: IntTuple) -> bool:
    """Identical nesting structure (leaf values ignored)."""
    stack = [(a, b)]
    while stack:
        x, y = stack.pop()
        tx, ty = isinstance(x, tuple), isinstance(y, tuple)
        if tx != ty or (tx and len(x) != len(y)):
            return False
        if tx:
            stack.extend(zip(x, y))
    return True


def zip_leaves(shape: IntTuple, stride: IntTuple) -> Iterator[Tuple[int, int]]:
    """(shape leaf, stride leaf) pairs in colex order; raises if the trees differ."""
    if not congruent(shape, stride):
        raise ShapeMismatch("shape and stride not congruent")
    return zip(leaves(shape), leaves(stride))


def decode(index: int, shape: IntTuple) -> Tuple[int, ...]:
    """Linear index -> flat digits (first leaf fastest)."""
    out = []
    for extent in leaves(shape):
        index, digit = divmod(index, extent)
        out.append(digit)
    return tuple(out)


def encode(digits, shape: IntTuple) -> int:
    """Flat digits -> linear index (inverse of :func:`decode`)."""
    total, weight = 0, 1
    for digit, extent in zip(digits, leaves(shape)):
        total += digit * weight
        weight *= extent
    return total


def format_tuple(t: IntTuple) -> str:
    """``(a,(b,c))`` with no spaces; a 1-tuple prints as ``(a)``."""
    return str(t) if isinstance(t, int) else "(" + ",".join(map(format_tuple, t)) + ")"


_TOKEN = re.compile(r"\d+|.")


def parse_tuple(text: str) -> IntTuple:
    """Text -> IntTuple. Spaces and tabs are ignored; empty tuples, dangling commas and trailing
    characters are errors."""
    body = text.replace(" ", "").replace("\t", "")
    stack: list = []          # open tuples being filled
    result = None
    want_item = True          # True after "(" or ",": an item must follow
    for m in _TOKEN.finditer(body):
        tok = m.group()
        if result is not None:
            raise ParseError(f"trailing characters in tuple: {body[m.start():]!r}")
        if tok == "(":
            if not want_item:
                raise ParseError(f"unexpected character {tok!r} in tuple")
            stack.append([])
            continue
        if tok.isdigit():
            if not want_item:
                raise ParseError(f"unexpected character {tok[0]!r} in tuple")
            item = int(tok)
        elif tok in ",)":
            if want_item or not stack:
                raise ParseError("empty tuple" if tok == ")" and stack and not stack[-1]
                                 else f"expected integer at {body[m.start():]!r}")
            if tok == ",":
                want_item = True
                continue
            item = tuple(stack.pop())
        else:
            if want_item:
                raise ParseError(f"expected integer at {body[m.start():]!r}")
            raise ParseError(f"unexpected character {tok!r} in tuple")
        if stack:
            stack[-1].append(item)
            want_item = False
        else:
            result = item
    if stack:
        raise ParseError("unterminated tuple")
    if result is None:
        raise ParseError("unexpected end of tuple")
    return result
