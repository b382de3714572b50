"""Nested non-negative integer tuples -- the shape and stride trees of layouts.

An IntTuple is an ``int`` or a ``tuple`` of IntTuples. A linear index is split over the leaves
colexicographically (leftmost leaf fastest). Same functions and meaning as
/root/reference/pkg/src/tilesynth/inttuple.py:1-143; here the tree walks are iterative (explicit
stacks), the parser is a token-driven state machine, and printing/congruence work on Python's own
tuple ``repr``.
"""
from __future__ import annotations

import math
import re
from typing import Tuple, Union

from .errors import IntegerOverflow, ParseError, ShapeMismatch

IntTuple = Union[int, Tuple["IntTuple", ...]]
INT64_MAX = (1 << 63) - 1

_WORD = re.compile(r"-?\w+")
_TOKENS = re.compile(r"\d+|.", re.S)


def is_int(t):
    return isinstance(t, int)


def leaves(t):
    """The leaves left to right (= colex digit order)."""
    if isinstance(t, int):
        return (t,)
    out, todo = [], [t]
    while todo:
        node = todo.pop()
        if isinstance(node, tuple):
            todo.extend(node[::-1])
        else:
            out.append(node)
    return tuple(out)


flatten = leaves


def validate(t, *, min_leaf=0):
    """Every leaf must be an int in [min_leaf, 2^63); the first offender (left to right) raises."""
    todo = [t]
    while todo:
        node = todo.pop()
        if isinstance(node, tuple):
            todo.extend(node[::-1])
        elif not isinstance(node, int):
            raise ShapeMismatch(f"{type(node).__name__} is neither an int nor a tuple")
        elif node < min_leaf:
            raise ShapeMismatch(f"{node} is below the smallest allowed leaf {min_leaf}")
        elif node > INT64_MAX:
            raise IntegerOverflow(f"{node} does not fit in 64 bits")


def congruent(a, b):
    """Same nesting: the ``repr`` strings agree once the leaf words are erased."""
    return _WORD.sub("", repr(a)) == _WORD.sub("", repr(b))


def size(t):
    return t if isinstance(t, int) else math.prod(leaves(t))


def depth(t):
    if isinstance(t, int):
        return 0
    return 1 + max(map(depth, t), default=0)


def zip_leaves(shape, stride):
    """(shape leaf, stride leaf) pairs in colex order; the trees must be congruent."""
    if not congruent(shape, stride):
        raise ShapeMismatch(f"{shape!r} and {stride!r} do not nest alike")
    return iter(tuple(zip(leaves(shape), leaves(stride))))


def decode(index, shape):
    """Linear index -> flat digits over the leaves (first leaf fastest)."""
    digits = []
    for extent in leaves(shape):
        index, digit = divmod(index, extent)
        digits.append(digit)
    return tuple(digits)


def encode(digits, shape):
    """Flat digits -> linear index (inverse of :func:`decode`), Horner from the slowest leaf."""
    index = 0
    for digit, extent in reversed(tuple(zip(digits, leaves(shape)))):
        index = index * extent + digit
    return index


def format_tuple(t):
    """``((2,4),8)`` style: Python's repr without blanks or the 1-tuple trailing comma."""
    return repr(t).replace(" ", "").replace(",)", ")")


def parse_tuple(text):
    """Inverse of :func:`format_tuple`; blanks and tabs are ignored, anything else malformed is a
    ParseError (empty groups, dangling commas, unbalanced parentheses, trailing text)."""
    groups = [[]]          # innermost open group last; groups[0] collects the single result
    expect_item = True     # an integer or '(' must come next
    for tok in _TOKENS.findall(text.replace(" ", "").replace("\t", "")):
        if expect_item:
            if tok == "(":
                groups.append([])
            elif tok.isdigit():
                groups[-1].append(int(tok))
                expect_item = False
            else:
                raise ParseError(f"expected an integer or '(' but found {tok!r}")
        elif len(groups) > 1 and tok == ",":
            expect_item = True
        elif len(groups) > 1 and tok == ")":
            closed = tuple(groups.pop())
            groups[-1].append(closed)
        else:
            raise ParseError(f"unexpected {tok!r} after a complete element")
    if expect_item or len(groups) > 1:
        raise ParseError("tuple text ends before it is complete")
    return groups[0][0]
